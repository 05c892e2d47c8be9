"""Benchmark harness over the GPU engine: seeded test matrices, the matrix suite, and the
flat CSV schema of the reference's bench module (reference
`pfexpm/bench.py`).

Each row times one engine call after a discarded warm-up, reporting the median of
`timing_repeats` runs:
  * t_para_ms  the slowest pole pair, from the CUDA events the engine reports per pair
               (`ExpResult.per_term_times`);
  * t_total_ms the call's wall clock (staging, kernels, the reduction, any NCCL reduce);
  * t_seq_ms   the host eigendecomposition that the error column is measured against.

Error convention (reference bench.py:15-17): absolute 2-norm error when the spectral
estimate is nonpositive, relative to ||exp(A)||_2 when positive eigenvalues are present;
vector norms in action mode.

CSV: `CSV_HEADER` is the reference's schema byte for byte.  Rows that also record how
many GPUs served the run are written under the versioned header `CSV_HEADER_V2` (one
extra trailing column, `devices`) to a separate file, so v1 consumers keep working;
`parse_csv` reads both.
"""
from __future__ import annotations

import csv
import math
import statistics
import time
from dataclasses import dataclass, field

import numpy as np

from .engine import MODE_ACTION, MODE_FULL, POSITIVE_FUZZ, ExpOptions, matexp_action, matexp_full, matexp_shifted
from .errors import BadSpec, ParseError
from .linalg import HermitianMatrix, SpectralBounds, gershgorin_bounds
from . import workloads

__all__ = [
    "CSV_HEADER",
    "CSV_HEADER_V2",
    "FAMILY_LAP1D",
    "FAMILY_LAP2D",
    "FAMILY_RANDOM",
    "BenchRecord",
    "MatrixSpec",
    "emit_csv",
    "gen_matrix",
    "parse_csv",
    "run_matrix_suite",
]

FAMILY_LAP1D = "lap1d"
FAMILY_LAP2D = "lap2d"
FAMILY_RANDOM = "random"
FAMILIES = (FAMILY_LAP1D, FAMILY_LAP2D, FAMILY_RANDOM)

_COLUMNS = ("family", "d", "n", "mode", "shift", "seed", "trial", "error", "error_kind", "t_seq_ms", "t_para_ms",
            "t_total_ms", "bound")
CSV_HEADER = ",".join(_COLUMNS)
CSV_HEADER_V2 = CSV_HEADER + ",devices"

ERROR_ABSOLUTE = "absolute"
ERROR_RELATIVE = "relative"


def _is_int(x) -> bool:
    return isinstance(x, int) and not isinstance(x, bool)


@dataclass(frozen=True)
class MatrixSpec:
    """Family, dimension, spectrum range (random family only) and seed of one test matrix."""

    family: str
    d: int
    spectrum_range: tuple | None = None
    seed: int = 0

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise BadSpec(f"unknown family {self.family!r}; families are {FAMILIES}")
        if not _is_int(self.d) or self.d < 1:
            raise BadSpec(f"d must be a positive integer, got {self.d!r}")
        if self.family == FAMILY_LAP2D and math.isqrt(self.d) ** 2 != self.d:
            raise BadSpec(f"lap2d is an m x m grid: d must be a perfect square, got {self.d}")
        if self.spectrum_range is not None:
            if self.family != FAMILY_RANDOM:
                raise BadSpec(f"spectrum_range applies to the random family only, not {self.family}")
            lo, hi = self.spectrum_range
            if not lo <= hi:
                raise BadSpec(f"spectrum_range needs lo <= hi, got {self.spectrum_range}")
        if not _is_int(self.seed) or self.seed < 0:
            raise BadSpec(f"seed must be a nonnegative integer, got {self.seed!r}")

    @property
    def grid_m(self) -> int:
        if self.family != FAMILY_LAP2D:
            raise BadSpec("grid_m is defined for the lap2d family only")
        return math.isqrt(self.d)


@dataclass(frozen=True)
class BenchRecord:
    """One CSV row; durations in milliseconds (medians over the timing repeats)."""

    spec: MatrixSpec
    n: int
    mode: str
    shift: float | None
    trial: int
    error: float
    error_kind: str
    t_seq: float
    t_para: float
    t_total: float
    bound: float | None
    devices: int = 1
    per_term_times: tuple = field(default=(), compare=False)

    def __post_init__(self):
        if not self.error >= 0.0:
            raise BadSpec(f"error must be >= 0, got {self.error!r}")
        if self.error_kind not in (ERROR_ABSOLUTE, ERROR_RELATIVE):
            raise BadSpec(f"error_kind must be absolute or relative, got {self.error_kind!r}")
        if self.mode not in (MODE_FULL, MODE_ACTION):
            raise BadSpec(f"mode must be full or action, got {self.mode!r}")
        if self.t_para > self.t_total:  # the slowest pair is inside the call's wall time
            raise BadSpec(f"t_para {self.t_para} exceeds t_total {self.t_total}")
        if not _is_int(self.devices) or self.devices < 1:
            raise BadSpec(f"devices must be a positive integer, got {self.devices!r}")


def _stencil_1d(d: int) -> np.ndarray:
    return np.diag(np.full(d, -2.0)) + np.diag(np.ones(d - 1), 1) + np.diag(np.ones(d - 1), -1)


def gen_matrix(spec: MatrixSpec, trial: int = 0) -> HermitianMatrix:
    """The test matrix of (spec, trial); deterministic.  Random family: the seeded recipe of
    reference bench.gen_matrix (bench.py:162-182), shared with `workloads`."""
    if spec.family == FAMILY_LAP1D:
        return HermitianMatrix(_stencil_1d(spec.d))
    if spec.family == FAMILY_LAP2D:
        T, eye = _stencil_1d(spec.grid_m), np.eye(spec.grid_m)
        return HermitianMatrix(np.kron(T, eye) + np.kron(eye, T))
    if spec.spectrum_range is None:
        raise BadSpec("the random family needs a spectrum_range")
    lo, hi = spec.spectrum_range
    A, lam_lo, lam_hi = workloads.random_real_symmetric(spec.d, lo, hi, spec.seed, trial)
    return HermitianMatrix(A, bounds=SpectralBounds(lam_lo, lam_hi, exact=True))


def _unit_vector(spec: MatrixSpec, trial: int) -> np.ndarray:
    return workloads.unit_vector(spec.d, spec.seed, trial)


def _exp_eigh(A: HermitianMatrix) -> np.ndarray:
    """exp(A) from the Hermitian eigendecomposition (the error column's reference value)."""
    w, U = np.linalg.eigh(A.entries)
    E = (U * np.exp(w)) @ U.conj().T
    return E.real if A.is_real() else E


def _positive_spectrum(A: HermitianMatrix) -> bool:
    b = A.bounds if A.bounds is not None else gershgorin_bounds(A)
    return b.hi > POSITIVE_FUZZ * max(1.0, abs(b.lo))


def _median_ms(fn, repeats: int):
    fn()  # warm-up
    out, ts = None, []
    for _ in range(repeats):
        t0 = time.perf_counter()
        out = fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return out, statistics.median(ts)


def _devices() -> int:
    try:
        import torch.distributed as dist

        return dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    except ImportError:  # pragma: no cover
        return 1


def _run_one(spec: MatrixSpec, n: int, mode: str, trial: int, threads, shift, repeats: int) -> BenchRecord:
    A = gen_matrix(spec, trial)
    v = _unit_vector(spec, trial) if mode == MODE_ACTION else None
    opts = ExpOptions(n=n, mode=mode, shift=shift, threads=threads)
    if shift is not None:
        call = lambda: matexp_shifted(A, opts, v=v)  # noqa: E731
    elif mode == MODE_ACTION:
        call = lambda: matexp_action(A, v, opts)  # noqa: E731
    else:
        call = lambda: matexp_full(A, opts)  # noqa: E731
    call()  # warm-up (first call also compiles nothing: the kernels are prebuilt)
    runs = [call() for _ in range(repeats)]
    res = runs[-1]
    t_para = statistics.median(r.t_para for r in runs) * 1e3
    t_total = statistics.median(r.t_total for r in runs) * 1e3

    if mode == MODE_ACTION:
        want, t_seq = _median_ms(lambda: _exp_eigh(A) @ v, repeats)
        err, scale = float(np.linalg.norm(res.value - want)), float(np.linalg.norm(want))
    else:
        want, t_seq = _median_ms(lambda: _exp_eigh(A), repeats)
        err, scale = float(np.linalg.norm(res.value - want, 2)), float(np.linalg.norm(want, 2))
    kind = ERROR_ABSOLUTE
    if _positive_spectrum(A):
        kind, err = ERROR_RELATIVE, err / scale

    bound = res.error_bound
    if bound is not None and res.bound_kind == "relative" and kind == ERROR_ABSOLUTE:
        # shifted run on a nonpositive spectrum: ||exp(A)||_2 = e^alpha <= e^c turns the
        # certified relative bound into an absolute one
        bound = bound * math.exp(res.c_applied)
    return BenchRecord(spec=spec, n=n, mode=mode, shift=res.c_applied, trial=trial, error=err, error_kind=kind,
                       t_seq=t_seq, t_para=t_para, t_total=t_total, bound=bound, devices=_devices(),
                       per_term_times=res.per_term_times)


def run_matrix_suite(spec_list, n_list, mode: str = MODE_FULL, trials: int = 1, threads="auto", shift=None,
                     timing_repeats: int = 3) -> list:
    """One BenchRecord per (spec, n, trial), run one after another (honest timings)."""
    if not _is_int(trials) or trials < 1:
        raise BadSpec(f"trials must be >= 1, got {trials!r}")
    if not _is_int(timing_repeats) or timing_repeats < 1:
        raise BadSpec(f"timing_repeats must be >= 1, got {timing_repeats!r}")
    return [_run_one(spec, n, mode, t, threads, shift, timing_repeats)
            for spec in spec_list for n in n_list for t in range(trials)]


def _f(x: float) -> str:
    return f"{x:.16e}"  # 17 significant digits: exact binary64 round trip


def emit_csv(records, path, devices: bool = False) -> None:
    """Write records under CSV_HEADER, or CSV_HEADER_V2 (with the devices column) when asked."""
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow((CSV_HEADER_V2 if devices else CSV_HEADER).split(","))
        for r in records:
            row = [r.spec.family, r.spec.d, r.n, r.mode, "none" if r.shift is None else _f(r.shift), r.spec.seed,
                   r.trial, _f(r.error), r.error_kind, _f(r.t_seq), _f(r.t_para), _f(r.t_total),
                   "" if r.bound is None else _f(r.bound)]
            if devices:
                row.append(r.devices)
            w.writerow(row)


def parse_csv(path) -> list:
    """Read a v1 or v2 bench CSV; the random family's spectrum range is not serialized."""
    out = []
    with open(path, "r", encoding="utf-8", newline="") as fh:
        reader = csv.DictReader(fh)
        hdr = reader.fieldnames
        if hdr not in (CSV_HEADER.split(","), CSV_HEADER_V2.split(",")):
            raise ParseError(f"unexpected CSV header {hdr!r}")
        for row in reader:
            spec = MatrixSpec(family=row["family"], d=int(row["d"]), seed=int(row["seed"]))
            out.append(BenchRecord(
                spec=spec, n=int(row["n"]), mode=row["mode"],
                shift=None if row["shift"] == "none" else float(row["shift"]), trial=int(row["trial"]),
                error=float(row["error"]), error_kind=row["error_kind"], t_seq=float(row["t_seq_ms"]),
                t_para=float(row["t_para_ms"]), t_total=float(row["t_total_ms"]),
                bound=None if row["bound"] == "" else float(row["bound"]),
                devices=int(row["devices"]) if "devices" in row else 1))
    return out
