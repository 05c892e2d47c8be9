"""CPU timing of the reference hot path — TEST / BASELINE INFRASTRUCTURE ONLY.

Used by bench.py's `cpu_baseline` leg and its `--impl reference` arm (nothing in the
product imports it).  It follows the reference's own timing discipline
(/root/reference/pkg/src/pfexpm/bench.py:196-205, `_median_timed`: one discarded warm-up,
then the median of the timed repeats) and BASELINE.md §3's thread settings:

    S1  procs=1      BLAS threads=1
    S2  procs=nproc  BLAS threads=1      (one process per work unit)
    S3  procs=1      BLAS threads=nproc

Run as a subprocess so that OPENBLAS_NUM_THREADS / OMP_NUM_THREADS are in the
environment BEFORE numpy (and OpenBLAS) load: setting them later is the
oversubscription trap SURVEY §4 measured at 40x.  Worker processes are `spawn`ed and
inherit that environment; each builds its inputs once, in its initializer, outside the
timed region.

What is timed (one "step" = every process runs one work unit; a unit is a bounded sample
of one eval, stated in `sample`):

    C1  reference matexp_action (baseline/_ref pfexpm, its public API), 40 evals per unit
    C3  reference matexp_action, 4 of the 512 matrices per unit
    C4  reference matexp_full with n = 2: exactly one of C4's 12 pair tasks
        (M = A + theta I, zgesv(M, I), aX + (aX)^H; engine.py:197,208,211-213), 1/12 eval
    C2  oracle restatement (the reference has no tridiagonal path):
        zgtsv per pair on one of the 16 RHS columns, all 12 pairs, 1/16 eval
    C5  oracle restatement: zgbsv (kl = ku = 512, 8 RHS) for one pole pair on the leading
        1/8 of the rows (band LU work is linear in the rows), 1/64 eval

C1/C3/C4 run the unmodified reference package from baseline/_ref when it is importable
(kind "reference"), else the restatement oracle/restate.py, which reproduces the
reference bit-for-bit (kind "port").  C2/C5 are always "port".

    python -m oracle.cpu_timer --workload C4 --procs 1 --blas 16 --steps 5 --warmup 1
prints one JSON line: {"value": evals/s (median step), ...}.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
C5_ROWS_FRAC = 8

_STATE = {}


def _have_reference() -> bool:
    return os.path.isdir(os.path.join(REF, "pfexpm"))


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import pfexpm  # noqa: WPS433 - the unmodified reference package

    return pfexpm


def unit_evals(name: str) -> float:
    return {"C1": 40.0, "C3": 4.0, "C4": 1.0 / 12.0, "C2": 1.0 / 16.0, "C5": 1.0 / 64.0}[name]


def describe(name: str, kind: str) -> str:
    who = "reference pfexpm (baseline/_ref) public API" if kind == "reference" else "oracle restatement"
    return {
        "C1": f"40 C1 evals per unit via {who} matexp_action (threads=1)",
        "C3": f"4 of the 512 C3 matrices per unit via {who} matexp_action (threads=1)",
        "C4": f"one of the 12 C4 pair tasks per unit (zgesv d=4096 with I, aX+(aX)^H) via {who}"
              + (" matexp_full n=2" if kind == "reference" else ""),
        "C2": "one of the 16 C2 RHS columns per unit, all 12 pairs, zgtsv (oracle restatement)",
        "C5": f"one of the 8 C5 pole pairs per unit, zgbsv kl=ku=512, 8 RHS, leading 1/{C5_ROWS_FRAC} of the rows "
              "(oracle restatement)",
    }[name]


def _init(name: str, kind: str):
    """Build the inputs once per process (outside the timed region)."""
    sys.path.insert(0, ROOT)
    import numpy as np

    from paper_2306_16778_b200 import workloads as W

    st = {"name": name, "kind": kind, "i": 0}
    if name == "C1":
        A, v, (lo, hi) = W.c1_inputs()
        st["args"] = (A, v, lo, hi)
    elif name == "C3":
        st["mats"] = [(W.c3_matrix(b), W.c3_vector(b), W.c3_bounds(b)) for b in range(4)]
    elif name == "C4":
        A, (lo, hi) = W.c4_matrix()
        st["args"] = (A, lo, hi)
    elif name == "C2":
        d, o = W.c2_matrix()
        st["args"] = (d, o, W.c2_rhs())
    elif name == "C5":
        from oracle import restate

        band = W.c5_band()
        V = W.c5_rhs()
        nk = band.shape[1] // C5_ROWS_FRAC
        band = np.ascontiguousarray(band[:, :nk])
        st["args"] = (restate.sym_band_to_general(band), band.shape[0] - 1, V[:nk].astype(complex))
    if kind == "reference" and name in ("C1", "C3", "C4"):
        pf = _ref()
        if name == "C1":
            A, v, lo, hi = st["args"]
            st["H"] = pf.HermitianMatrix(A, bounds=pf.SpectralBounds(lo, hi, exact=True))
        elif name == "C4":
            A, lo, hi = st["args"]
            st["H"] = pf.HermitianMatrix(A, bounds=pf.SpectralBounds(lo, hi, exact=True))
        else:
            st["Hs"] = [(pf.HermitianMatrix(A, bounds=pf.SpectralBounds(b.lo, b.hi, exact=True)), v)
                        for A, v, b in st["mats"]]
    _STATE.clear()
    _STATE.update(st)


def _unit(_=None) -> float:
    """One work unit; returns the evals it represents."""
    import warnings

    import numpy as np

    st = _STATE
    name, kind = st["name"], st["kind"]
    warnings.simplefilter("ignore")
    if name in ("C1", "C3", "C4") and kind == "reference":
        pf = _ref()
        if name == "C1":
            opts = pf.ExpOptions(n=16, mode="action", threads=1)
            for _ in range(40):
                pf.matexp_action(st["H"], st["args"][1], opts)
        elif name == "C3":
            opts = pf.ExpOptions(n=20, mode="action", threads=1)
            for H, v in st["Hs"]:
                pf.matexp_action(H, v, opts)
        else:
            pf.matexp_full(st["H"], pf.ExpOptions(n=2, mode="full", threads=1))
        return unit_evals(name)
    from oracle import restate

    if name == "C1":
        A, v = st["args"][:2]
        for _ in range(40):
            restate.run_tasks_dense(A, v, 16)
    elif name == "C3":
        for A, v, _b in st["mats"]:
            restate.run_tasks_dense(A, v, 20)
    elif name == "C4":
        A = st["args"][0]
        th, co = restate.pairs(24)
        X = np.linalg.solve(A + th[st["i"] % 12] * np.eye(A.shape[0]), np.eye(A.shape[0], dtype=complex))
        aX = co[st["i"] % 12] * X
        _ = aX + aX.conj().T
    elif name == "C2":
        d, o, V = st["args"]
        restate.tridiag_action(d, o, V, 24, cols=[st["i"] % 16])
    elif name == "C5":
        import scipy.linalg.lapack as lapack

        base, kb, B = st["args"]
        th, _co = restate.pairs(16)
        ab = base.copy()
        ab[2 * kb, :] += th[st["i"] % 8]
        lapack.zgbsv(kb, kb, ab, B, overwrite_ab=1)
    st["i"] += 1
    return unit_evals(name)


def run(name: str, procs: int, steps: int, warmup: int, kind: str):
    """Median-of-steps throughput (evals/s) after `warmup` discarded steps."""
    times = []
    evals = 0.0
    if procs <= 1:
        _init(name, kind)
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            evals = _unit()
            dt = time.perf_counter() - t0
            if it >= warmup:
                times.append(dt)
    else:
        import multiprocessing as mp

        ctx = mp.get_context("spawn")
        with ctx.Pool(procs, initializer=_init, initargs=(name, kind)) as pool:
            pool.map(_noop, range(procs))  # every worker initialised before timing
            for it in range(warmup + steps):
                t0 = time.perf_counter()
                evals = sum(pool.map(_unit, range(procs), chunksize=1))
                dt = time.perf_counter() - t0
                if it >= warmup:
                    times.append(dt)
    med = statistics.median(times)
    return evals / med, med, times


def _noop(_):
    return 0


def blas_info():
    try:
        import threadpoolctl

        return [f"{i['internal_api']} {i['version']} threads={i['num_threads']}"
                for i in threadpoolctl.threadpool_info() if i.get("user_api") == "blas"]
    except Exception:  # pragma: no cover
        return []


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", required=True, choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--procs", type=int, default=1)
    ap.add_argument("--blas", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--kind", choices=["auto", "reference", "port"], default="auto")
    a = ap.parse_args()
    if os.environ.get("OPENBLAS_NUM_THREADS") != str(a.blas):
        # re-exec with the BLAS thread count in the environment before numpy loads
        env = dict(os.environ, OPENBLAS_NUM_THREADS=str(a.blas), OMP_NUM_THREADS=str(a.blas),
                   MKL_NUM_THREADS=str(a.blas))
        os.execvpe(sys.executable, [sys.executable, "-m", "oracle.cpu_timer", *sys.argv[1:]], env)
    kind = a.kind
    if kind == "auto":
        kind = "reference" if (a.workload in ("C1", "C3", "C4") and _have_reference()) else "port"
    value, med, times = run(a.workload, a.procs, a.steps, a.warmup, kind)
    print(json.dumps({
        "workload": a.workload, "value": value, "unit": "evals/s", "median_step_s": med, "step_s": times,
        "procs": a.procs, "blas_threads": a.blas, "cores": a.procs * a.blas, "steps": a.steps, "warmup": a.warmup,
        "kind": kind, "sample": describe(a.workload, kind) + f"; {a.procs} process(es) x {a.blas} BLAS thread(s)",
        "unit_evals": unit_evals(a.workload), "nproc": os.cpu_count(), "blas": blas_info(),
    }), flush=True)


if __name__ == "__main__":
    main()
