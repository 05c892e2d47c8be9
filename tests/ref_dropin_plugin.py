"""pytest plugin (test infrastructure): loaded with `-p tests.ref_dropin_plugin` into a run of
the REFERENCE's own test files, it installs the libpfx.so drop-in
(paper_2306_16778_b200/dropin.py) into the reference engine before any test runs, counts the
calls that reached the library, and prints the count at the end of the session."""
import pfexpm.engine as _engine

from paper_2306_16778_b200 import dropin

_CALLS = [0]


def pytest_configure(config):
    inner = dropin.make_run_tasks(_engine)

    def counted(A, v, opts):
        _CALLS[0] += 1
        return inner(A, v, opts)

    _engine._run_tasks = counted


def pytest_sessionfinish(session, exitstatus):
    print(f"\nPFX_DROPIN_CALLS={_CALLS[0]}")
