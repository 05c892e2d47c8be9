"""paper_2306_16778_b200.bench: the harness around the hot path, mirroring
the reference's bench module tests (reference tests/test_bench.py) for the matrix suite and
the CSV schema."""
import numpy as np
import pytest

from paper_2306_16778_b200 import bench as B
from paper_2306_16778_b200.errors import BadSpec, ParseError


class TestSpec:
    def test_valid(self):
        B.MatrixSpec("lap1d", 5)
        B.MatrixSpec("lap2d", 16)
        B.MatrixSpec("random", 8, (-3.0, 0.0), seed=2)

    @pytest.mark.parametrize("kw", [dict(family="nope", d=4), dict(family="lap1d", d=0), dict(family="lap1d", d=2.0),
                                    dict(family="lap2d", d=15), dict(family="lap1d", d=4, spectrum_range=(-1, 0)),
                                    dict(family="random", d=4, spectrum_range=(1.0, 0.0)),
                                    dict(family="lap1d", d=4, seed=-1), dict(family="lap1d", d=4, seed=True)])
    def test_invalid(self, kw):
        with pytest.raises(BadSpec):
            B.MatrixSpec(**kw)


class TestGenerators:
    def test_lap1d_stencil(self):
        A = B.gen_matrix(B.MatrixSpec("lap1d", 3)).entries
        assert np.array_equal(A, [[-2, 1, 0], [1, -2, 1], [0, 1, -2]])

    @pytest.mark.parametrize("d", [1, 7, 40])
    def test_lap1d_spectrum(self, d):
        w = np.linalg.eigvalsh(B.gen_matrix(B.MatrixSpec("lap1d", d)).entries)
        assert w.min() > -4.0 and w.max() < 0.0

    def test_lap2d_is_kronecker_sum(self):
        m = 4
        w = np.linalg.eigvalsh(B.gen_matrix(B.MatrixSpec("lap2d", m * m)).entries)
        w1 = -2.0 + 2.0 * np.cos(np.arange(1, m + 1) * np.pi / (m + 1))
        assert np.allclose(np.sort(w), np.sort(np.add.outer(w1, w1).ravel()))

    def test_random_spectrum_and_determinism(self):
        s = B.MatrixSpec("random", 30, (-20.0, -1.0), seed=5)
        A1, A2, A3 = B.gen_matrix(s, 0), B.gen_matrix(s, 0), B.gen_matrix(s, 1)
        assert np.array_equal(A1.entries, A2.entries) and not np.array_equal(A1.entries, A3.entries)
        w = np.linalg.eigvalsh(A1.entries)
        assert A1.bounds.exact and abs(w[0] - A1.bounds.lo) < 1e-10 and abs(w[-1] - A1.bounds.hi) < 1e-10

    def test_random_needs_range(self):
        with pytest.raises(BadSpec):
            B.gen_matrix(B.MatrixSpec("random", 4))


def _rec(**kw):
    base = dict(spec=B.MatrixSpec("lap1d", 6), n=16, mode="full", shift=None, trial=0, error=1e-16,
                error_kind="absolute", t_seq=1.0, t_para=0.25, t_total=0.5, bound=3e-5)
    base.update(kw)
    return B.BenchRecord(**base)


class TestRecords:
    @pytest.mark.parametrize("kw", [dict(error=-1.0), dict(error_kind="weird"), dict(mode="x"),
                                    dict(t_para=2.0, t_total=1.0), dict(devices=0)])
    def test_invalid(self, kw):
        with pytest.raises(BadSpec):
            _rec(**kw)


class TestCsv:
    def test_header_is_the_reference_schema(self):
        assert B.CSV_HEADER == ("family,d,n,mode,shift,seed,trial,error,error_kind,"
                                "t_seq_ms,t_para_ms,t_total_ms,bound")
        assert B.CSV_HEADER_V2 == B.CSV_HEADER + ",devices"

    def test_roundtrip_v1_and_v2(self, tmp_path):
        recs = [_rec(), _rec(shift=-1.5, trial=1, bound=None, error_kind="relative", mode="action"),
                _rec(devices=4)]
        p1, p2 = tmp_path / "a.csv", tmp_path / "b.csv"
        B.emit_csv(recs, p1)
        B.emit_csv(recs, p2, devices=True)
        assert p1.read_text().splitlines()[0] == B.CSV_HEADER
        assert p2.read_text().splitlines()[0] == B.CSV_HEADER_V2
        back1, back2 = B.parse_csv(p1), B.parse_csv(p2)
        assert [r.devices for r in back1] == [1, 1, 1]  # v1 does not carry it
        assert back2 == recs
        assert [(r.error, r.t_para, r.bound) for r in back1] == [(r.error, r.t_para, r.bound) for r in recs]

    def test_uncertified_bound_written_empty(self, tmp_path):
        p = tmp_path / "c.csv"
        B.emit_csv([_rec(bound=None)], p)
        assert p.read_text().splitlines()[1].endswith(",")

    def test_header_only_and_bad_header(self, tmp_path):
        p = tmp_path / "d.csv"
        B.emit_csv([], p)
        assert p.read_text() == B.CSV_HEADER + "\n"
        assert B.parse_csv(p) == []
        q = tmp_path / "e.csv"
        q.write_text("family,d\nlap1d,3\n")
        with pytest.raises(ParseError):
            B.parse_csv(q)


@pytest.mark.gpu
class TestSuiteGpu:
    def test_lap1d_full_within_bound(self):
        # lap1d: Gershgorin [-4, 0], rho = 2, so n > 4 admits the certified bound
        # (orders where the truncation error, not the 2n-term rounding floor, dominates)
        recs = B.run_matrix_suite([B.MatrixSpec("lap1d", 24)], [12, 16], timing_repeats=2)
        assert len(recs) == 2
        for r in recs:
            assert r.error_kind == "absolute" and r.bound is not None and r.error <= r.bound
            assert 0.0 <= r.t_para <= r.t_total and len(r.per_term_times) == r.n // 2

    def test_action_and_random_shifted(self):
        # the error column is the method's approximation error against eigh, within the bound
        ra = B.run_matrix_suite([B.MatrixSpec("random", 40, (-5.0, 0.0), seed=1)], [16], mode="action",
                                trials=2, timing_repeats=1)
        assert len(ra) == 2
        assert all(r.bound is not None and r.error <= r.bound for r in ra)
        rs = B.run_matrix_suite([B.MatrixSpec("random", 40, (-5.0, 4.0), seed=2)], [16], shift="auto",
                                timing_repeats=1)
        r = rs[0]
        assert r.error_kind == "relative" and r.shift is not None and r.shift > 0.0
        assert r.error <= (r.bound if r.bound is not None else 1e-5)  # n = 16 truncation level
