"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container only (the reference is not present on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (all committed, all small):
  tables/n{N}.txt        roots.table_to_text(default_table(N)) for every even N in 2..64
                         (reference pkg/src/pfexpm/roots.py:315-318, 349-357)
  tables_f8.npz          thetas_f8()/coeffs_f8() per N (roots.py:222-226), complex128
  dense_cases.npz        inputs + reference outputs of engine.matexp_action/_full/_shifted
                         (engine.py:254-320) on small seeded matrices, plus config C1
  c3_head.npz            reference matexp_action outputs for the first 4 matrices of C3
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import pfexpm  # noqa: E402  (the reference)
from pfexpm import (  # noqa: E402
    ExpOptions, HermitianMatrix, MatrixSpec, SpectralBounds, default_table,
    gen_matrix, matexp_action, matexp_full, matexp_shifted, table_to_text, exp_oracle,
)
from pfexpm.bench import _unit_vector  # noqa: E402

from paper_2306_16778_b200 import workloads as G  # noqa: E402  (seeded recipes)


def tables():
    f8 = {}
    for n in range(2, 65, 2):
        t = default_table(n)
        with open(os.path.join(HERE, "tables", f"n{n}.txt"), "w", newline="\n") as fh:
            fh.write(table_to_text(t))
        f8[f"theta_{n}"] = t.thetas_f8()
        f8[f"coef_{n}"] = t.coeffs_f8()
    np.savez_compressed(os.path.join(HERE, "tables_f8.npz"), **f8)


def _complex_negative(d, seed):
    # same recipe as reference tests/test_engine.py:63-77
    rng = np.random.default_rng(seed)
    C = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    A = -(C @ C.conj().T) / d
    A = (A + A.conj().T) / 2.0
    w = np.linalg.eigvalsh(A)
    return HermitianMatrix(A, bounds=SpectralBounds(float(1.01 * w[0]), min(float(w[-1]), 0.0), exact=False))


def dense_cases():
    out = {}
    cases = []
    # (name, matrix, v or None, opts)
    spec = MatrixSpec("random", 128, (-50.0, 0.0), seed=0)
    A = gen_matrix(spec, 0)
    v = _unit_vector(spec, 0)
    cases.append(("c1", A, v, ExpOptions(n=16, mode="action", threads=1)))
    for d, n in ((7, 8), (33, 16), (64, 24)):
        sp = MatrixSpec("random", d, (-20.0, 0.0), seed=3)
        Ad = gen_matrix(sp, 1)
        vd = _unit_vector(sp, 1)
        cases.append((f"real_action_d{d}_n{n}", Ad, vd, ExpOptions(n=n, mode="action", threads=1)))
        cases.append((f"real_full_d{d}_n{n}", Ad, None, ExpOptions(n=n, mode="full", threads=1)))
    for d, n, seed in ((25, 16, 23), (40, 20, 11)):
        Ac = _complex_negative(d, seed)
        rng = np.random.default_rng(seed + 100)
        vc = rng.standard_normal(d) + 1j * rng.standard_normal(d)
        vr = rng.standard_normal(d)
        cases.append((f"cplx_action_d{d}_n{n}", Ac, vc, ExpOptions(n=n, mode="action", threads=1)))
        cases.append((f"cplx_action_realv_d{d}_n{n}", Ac, vr, ExpOptions(n=n, mode="action", threads=1)))
        cases.append((f"cplx_full_d{d}_n{n}", Ac, None, ExpOptions(n=n, mode="full", threads=1)))
    # complex v on a real matrix (reference tests/test_engine.py:260-267)
    Al = gen_matrix(MatrixSpec("lap1d", 12), 0)
    rng = np.random.default_rng(31)
    cases.append(("lap1d_cplxv_d12_n16", Al, rng.standard_normal(12) + 1j * rng.standard_normal(12),
                  ExpOptions(n=16, mode="action", threads=1)))
    # shifted (engine.py:283-320)
    As = gen_matrix(MatrixSpec("random", 30, (0.0, 3.0), seed=21), 0)
    cases.append(("shift_full_d30_n16", As, None, ExpOptions(n=16, shift="auto", threads=1)))
    vs = _unit_vector(MatrixSpec("random", 30, (0.0, 3.0), seed=21), 0)
    cases.append(("shift_action_d30_n16", As, vs, ExpOptions(n=16, mode="action", shift="auto", threads=1)))
    names = []
    for name, A, v, opts in cases:
        if opts.shift is not None:
            res = matexp_shifted(A, opts, v=v)
        elif v is None:
            res = matexp_full(A, opts)
        else:
            res = matexp_action(A, v, opts)
        out[f"{name}__A"] = A.entries
        if v is not None:
            out[f"{name}__v"] = np.asarray(v)
        out[f"{name}__n"] = np.int64(opts.n)
        out[f"{name}__mode"] = np.array(opts.mode)
        out[f"{name}__shift"] = np.array("none" if opts.shift is None else str(opts.shift))
        out[f"{name}__value"] = res.value
        out[f"{name}__c"] = np.float64(np.nan if res.c_applied is None else res.c_applied)
        E = exp_oracle(A)
        out[f"{name}__oracle"] = E @ v if v is not None else E
        names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "dense_cases.npz"), **out)


def c3_head(count=4):
    vals, ors = [], []
    for b in range(count):
        A, v = G.c3_matrix(b), G.c3_vector(b)
        H = HermitianMatrix(A, bounds=G.c3_bounds(b))
        res = matexp_action(H, v, ExpOptions(n=20, mode="action", threads=1))
        vals.append(res.value)
        ors.append(exp_oracle(H) @ v)
    np.savez_compressed(os.path.join(HERE, "c3_head.npz"), value=np.array(vals), oracle=np.array(ors))


if __name__ == "__main__":
    assert "reference" in pfexpm.__file__, pfexpm.__file__
    tables()
    dense_cases()
    c3_head()
    print("golden fixtures written")
