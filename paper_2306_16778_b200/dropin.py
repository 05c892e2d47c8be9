"""The drop-in: libpfx.so behind the UNMODIFIED reference package's own hot-path function.

The reference (`pfexpm`, arXiv 2306.16778) has no FFI; its hot path is the private
`pfexpm.engine._run_tasks(A, v, opts) -> (acc, per_task_times, t_total)`
(/root/reference/pkg/src/pfexpm/engine.py:178-230), called from `_matexp` (engine.py:241) and
`matexp_shifted` (engine.py:302).  `install(engine)` replaces that one function of a loaded
reference engine module with `make_run_tasks(engine)`, which keeps the reference's contract
line by line and sends the arithmetic to `pfx_expm_dense` (include/pfx.h) with host buffers:

  * table     default_table(opts.n) of the reference itself, pair representatives at even
              indices (engine.py:180-182,196);
  * v         shape (d,) else BadSpec (engine.py:186-189); real_path = A.is_real() and v real
              or absent (engine.py:185) -> float64 output, else complex128;
  * combine   2 Re(a y) / a y + conj(a) yc / aX + (aX)^H, ascending pair sum
              (engine.py:199-213,225-228) -- inside the library;
  * timings   per_term_times = per-pair device time (CUDA events), n/2 entries, so
              t_para = max(per_term_times) holds (engine.py:114-118); t_total = wall clock;
  * errors    status -> the reference's own exception classes (errors.py:4-61).

This is the module INTEGRATION.md §2-3 describes, runnable: tests/test_reference_dropin_gpu.py
installs it into the reference from baseline/_ref and runs the reference's own engine tests.
"""
from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _native


def make_run_tasks(engine):
    """A `_run_tasks(A, v, opts)` for the reference engine module `engine`."""
    errors = __import__(engine.__name__.rsplit(".", 1)[0] + ".errors", fromlist=["errors"])
    default_table = engine.default_table

    def _raise(status: int, what: str):
        msg = f"{what}: {_native.last_error()}"
        if status == 1:
            raise errors.SingularSystem(msg)
        if status == 2:
            raise errors.BadSpec(msg)
        raise errors.PfexpmError(msg)

    def _run_tasks(A, v, opts):
        table = default_table(opts.n)
        thetas = np.ascontiguousarray(table.thetas_f8()[0::2])
        coeffs = np.ascontiguousarray(table.coeffs_f8()[0::2])
        d = A.d
        action = v is not None
        real_path = A.is_real() and (not action or bool(np.isrealobj(v)))
        if action:
            vv = np.asarray(v)
            if vv.shape != (d,):
                raise errors.BadSpec(f"v must have shape ({d},), got {vv.shape}")
            vv = np.ascontiguousarray(vv, dtype=np.float64 if np.isrealobj(vv) else np.complex128)
        a = np.ascontiguousarray(A.entries.real) if A.is_real() else np.ascontiguousarray(A.entries)
        npairs = thetas.shape[0]
        ncols = d if not action else 1
        out = np.empty((d, ncols), dtype=np.float64 if real_path else np.complex128)
        ms = (ctypes.c_float * npairs)()
        t2 = thetas.view(np.float64)
        c2 = coeffs.view(np.float64)
        _native._torch()  # a CUDA device must be present: no CPU fallback
        t0 = time.perf_counter()
        st = _native.lib().pfx_expm_dense(
            _native.PFX_MEM_HOST, a.ctypes.data, int(np.iscomplexobj(a)), d, 1,
            vv.ctypes.data if action else None, int(action and np.iscomplexobj(vv)), 1 if action else 0, 0.0,
            _native._f64p(t2), _native._f64p(c2), npairs, out.ctypes.data, int(not real_path),
            ctypes.cast(ms, ctypes.POINTER(ctypes.c_float)), None,
        )
        t_total = time.perf_counter() - t0
        if st:
            _raise(st, "pfx_expm_dense")
        acc = out[:, 0] if action else out
        return acc, tuple(float(x) * 1e-3 for x in ms), t_total

    _run_tasks.__pfx_dropin__ = True
    return _run_tasks


def install(engine):
    """Replace engine._run_tasks by the libpfx.so drop-in; returns a callable that restores it."""
    original = engine._run_tasks
    engine._run_tasks = make_run_tasks(engine)

    def restore():
        engine._run_tasks = original

    return restore
