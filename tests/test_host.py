"""CPU: host-side logic — containers (matrix.hpp), the seeded input
generators against the reference generator and the survey's probe numbers,
and the byte model the roofline uses."""
import numpy as np
import pytest

import oracle
from paper_2011_06391_b200 import configs
from paper_2011_06391_b200 import fusedmm as F


# ----------------------------------------------------------- containers
def test_csr_from_coo_dedup_first_occurrence_order():
    # matrix.hpp:84-140: duplicates summed, storage order = first occurrence
    A = F.csr_from_coo([(0, 2, 1.0), (0, 0, 2.0), (0, 2, 3.0), (1, 1, 1.0)], 2, 3)
    assert A.row_ptr.tolist() == [0, 2, 3]
    assert A.col_idx.tolist() == [2, 0, 1]
    assert A.values.tolist() == [4.0, 2.0, 1.0]
    with pytest.raises(F.InvalidArgument):
        F.csr_from_coo([(0, 3, 1.0)], 2, 3)


def test_csr_roundtrip_property():
    # test_core.cpp:100-135
    rng = np.random.default_rng(11)
    for _ in range(30):
        m, n = int(rng.integers(1, 20)), int(rng.integers(1, 20))
        ent = [(int(rng.integers(0, m)), int(rng.integers(0, n)), float(rng.uniform(0.1, 2))) for _ in
               range(int(rng.integers(0, m * n + 1)))]
        A = F.csr_from_coo(ent, m, n)
        assert F.validate(A) is None
        exp = {}
        for r, c, v in ent:
            exp[(r, c)] = exp.get((r, c), 0.0) + v
        got = {(r, int(A.col_idx[p])): float(A.values[p]) for r in range(m)
               for p in range(A.row_ptr[r], A.row_ptr[r + 1])}
        assert set(got) == set(exp)
        for k in exp:
            assert got[k] == pytest.approx(exp[k], rel=1e-5)


def test_validate_and_stats():
    A = F.CsrMatrix(2, 2, np.array([0, 2, 1]), np.array([0, 1]))
    assert "monotone" in F.validate(A)
    A = F.CsrMatrix(1, 2, np.array([0, 2]), np.array([1, 1]))
    assert "duplicate" in F.validate(A)
    A = F.csr_from_coo([(0, v, 1.0) for v in range(1, 6)], 6, 6)  # star (test_core.cpp:83-90)
    s = F.stats(A)
    assert s.max_degree == 5 and s.avg_degree == pytest.approx(5 / 6)
    with pytest.raises(F.InvalidArgument):
        F.DenseMatrix(1, 2, [1.0, np.nan])  # test_core.cpp:138-141


# ----------------------------------------------------------- generators
def test_generators_are_deterministic():
    a = configs.config2(scale=10)
    b = configs.config2(scale=10)
    assert np.array_equal(a.A.col_idx, b.A.col_idx) and np.array_equal(a.X.data, b.X.data)


@pytest.mark.parametrize("cfg", [2, 3, 5])
def test_rmat_postprocessing_properties(cfg):
    w = configs.get(cfg, small=True)
    A = w.A
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_ptr))
    assert not np.any(rows == A.col_idx)  # self-loops dropped
    assert F.validate(A) is None  # sorted unique, in range
    key = set(zip(rows.tolist(), A.col_idx.tolist()))
    assert all((c, r) in key for r, c in key)  # symmetric
    for u in range(0, A.nrows, max(1, A.nrows // 50)):
        assert np.all(np.diff(A.row_cols(u)) > 0)


def test_config1_recipe():
    w = configs.config1(n=512)
    A = w.A
    assert np.all(np.diff(A.row_ptr) == 16)
    for u in range(512):
        c = A.row_cols(u)
        assert np.all(np.diff(c) > 0)
    assert A.values.min() >= 0 and A.values.max() < 1
    assert w.X.data.min() >= -1 and w.X.data.max() < 1


def test_config4_recipe():
    w = configs.config4(side=32)
    A = w.A
    deg = np.diff(A.row_ptr)
    assert deg.min() >= 2 and deg.max() <= 15
    assert abs(w.X.array[5 * 32 + 7, 0] - 7) < 0.1 and abs(w.X.array[5 * 32 + 7, 1] - 5) < 0.1


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built here")
def test_rmat_symmetrised_equals_reference_stream_postprocessed():
    # our generator == reference rmat_generate (rmat.hpp:24-61) + BASELINE's
    # post-processing (drop self-loops, symmetrise, dedup, sort)
    rp, cl, _ = oracle.ref_rmat(11, 8, 99)
    rows = np.repeat(np.arange(2048), np.diff(rp))
    keep = rows != cl
    r2 = np.concatenate([rows[keep], cl[keep]])
    c2 = np.concatenate([cl[keep], rows[keep]])
    key = np.unique(r2 * 2048 + c2)
    A = configs.rmat_sym(11, 8, 99)
    assert np.array_equal(A.col_idx, key % 2048)
    assert np.array_equal(np.diff(A.row_ptr), np.bincount(key // 2048, minlength=2048))


# ------------------------------------------------- pins at full size (survey)
@pytest.mark.slow
def test_full_size_graphs_match_survey_probe():
    # SURVEY.md §8(d) [probe] numbers, produced with the reference generator
    w1 = configs.config1()
    assert w1.A.nnz() == 262144 and w1.alg_bytes() == 73_531_400
    w2 = configs.config2()
    deg = np.diff(w2.A.row_ptr)
    assert w2.A.nnz() == 31_398_704 and int(deg.max()) == 64_782 and int((deg == 0).sum()) == 402_719
    assert w2.alg_bytes() == 17_077_669_576
    w3 = configs.config3(iters=1)
    deg = np.diff(w3.A.row_ptr)
    assert w3.A.nnz() == 32_417_756 and int(deg.max()) == 62_004 and int((deg == 0).sum()) == 1_048_972
    assert w3.alg_bytes() == 4_698_523_512
    w4 = configs.config4()
    assert w4.A.nnz() == 25_157_628 and int(np.diff(w4.A.row_ptr).max()) == 15
    assert w4.alg_bytes() == 402_554_840


def test_bulk_mt19937_64_matches_std():
    # the vectorised generator behind the parallel R-MAT stream is
    # bit-identical to std::mt19937_64 across uneven block boundaries
    import ctypes as C
    from paper_2011_06391_b200 import _lib
    G = _lib.gen()
    G.fmmgen_mt64_check.restype = C.c_int64
    G.fmmgen_mt64_check.argtypes = [C.c_uint64, C.c_int64]
    for seed in (0, 1, 4, 5489, 2**63 + 7):
        assert G.fmmgen_mt64_check(seed, 300_000) == 0


def test_parity_rejects_non_finite_mismatch():
    """a NaN (or a finite/non-finite mismatch) in a GPU row must
    fail the tolerance gate; identical non-finite values (the AMAX identity
    -inf of an empty row) must not."""
    from tests.parity import check_tolerance
    A = F.CsrMatrix(3, 3, np.array([0, 1, 1, 2]), np.array([1, 0]), None)
    X = F.DenseMatrix(3, 2, np.ones(6, np.float32))
    spec = F.OpSpec(F.Vop.MUL, F.Rop.NOOP, F.Sop.NOOP, F.Mop.MUL, F.Aop.AMAX)
    Zr = oracle.oracle_fused_mm(A, X, X, spec)
    assert np.isneginf(Zr[1]).all()  # empty row: the AMAX identity
    check_tolerance(Zr.copy(), Zr, A, X, X, spec)  # identical incl. -inf: passes
    bad = Zr.copy()
    bad[0, 1] = np.nan
    with pytest.raises(AssertionError):
        check_tolerance(bad, Zr, A, X, X, spec)
    bad = Zr.copy()
    bad[1, 0] = 0.0  # finite where the oracle has -inf
    with pytest.raises(AssertionError):
        check_tolerance(bad, Zr, A, X, X, spec)
    e = oracle.row_errors(np.array([[np.nan, 1.0]]), np.array([[np.nan, 1.0]]))
    assert e[0] == 0.0


# ----------------------------------------------------------- work lists
def _plan_pieces(A, rb=0, re=None):
    import ctypes as C
    from paper_2011_06391_b200 import _lib
    re = A.nrows if re is None else re
    L = _lib.lib()
    rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.col_idx, dtype=np.int64)
    p64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))
    chunk, ns, nb, npc = (C.c_int64() for _ in range(4))
    assert L.fmm_plan_pieces(A.nrows, A.ncols, p64(rp), p64(ci), rb, re, C.byref(chunk), C.byref(ns), C.byref(nb),
                             C.byref(npc), None, 0) == 0
    out = np.zeros((max(npc.value, 1), 4), dtype=np.int64)
    assert L.fmm_plan_pieces(A.nrows, A.ncols, p64(rp), p64(ci), rb, re, None, None, None, None, p64(out),
                             npc.value) == 0
    return chunk.value, ns.value, nb.value, out[:npc.value]


def _heavy_graph(seed, n=8192):
    rng = np.random.default_rng(seed)
    deg = np.zeros(n, dtype=np.int64)
    deg[rng.choice(n, 30, replace=False)] = rng.integers(64, 2500, 30)
    light = rng.choice(n, n // 3, replace=False)
    deg[light] = np.where(deg[light] == 0, rng.integers(1, 10, light.size), deg[light])
    row_ptr = np.concatenate([[0], np.cumsum(deg)])
    cols = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in deg if k > 0])
    return F.CsrMatrix(n, n, row_ptr, cols, None)


def test_plan_pieces_fixed_chunks_cover_split_rows(monkeypatch):
    """Without column bands (small n) only rows longer than the chunk size are
    cut, into consecutive chunk-size pieces that cover the row exactly."""
    monkeypatch.setenv("FMM_BANDS", "0")
    monkeypatch.setenv("FMM_CHUNK", "256")
    A = _heavy_graph(1)
    chunk, ns, nb, pc = _plan_pieces(A)
    deg = np.diff(A.row_ptr)
    assert chunk == 256 and nb == 0 and ns == int((deg > 256).sum())
    for r in np.unique(pc[:, 0]):
        mine = pc[pc[:, 0] == r]
        mine = mine[np.argsort(mine[:, 1])]
        assert mine[0, 1] == 0 and (mine[:-1, 1] + mine[:-1, 2] == mine[1:, 1]).all()
        assert mine[:, 2].sum() == deg[r] and (mine[:-1, 2] == 256).all() and mine[-1, 2] <= 256


def test_plan_pieces_column_bands(monkeypatch):
    """Column bands: rows of min_deg+ edges are cut where their (ascending)
    columns cross a band boundary once a piece has min_len edges; pieces never
    exceed the chunk size, cover each row exactly, and launch band-major."""
    monkeypatch.setenv("FMM_BAND_COLS", "64")
    monkeypatch.setenv("FMM_BAND_MINDEG", "64")
    monkeypatch.setenv("FMM_BAND_MINLEN", "4")
    monkeypatch.setenv("FMM_CHUNK", "256")
    A = _heavy_graph(2)
    deg = np.diff(A.row_ptr)
    chunk, ns, nb, pc = _plan_pieces(A)
    assert ns == int((deg >= 64).sum()) and nb == ns and len(pc) > ns
    assert (np.diff(pc[:, 3]) >= 0).all()  # band-major launch order
    for r in np.unique(pc[:, 0]):
        mine = pc[pc[:, 0] == r]
        mine = mine[np.argsort(mine[:, 1])]
        assert mine[0, 1] == 0 and (mine[:-1, 1] + mine[:-1, 2] == mine[1:, 1]).all()
        assert mine[:, 2].sum() == deg[r] and (mine[:, 2] <= chunk).all()
        cols = A.col_idx[A.row_ptr[r]:A.row_ptr[r + 1]]
        for e0, ln, band in mine[:, 1:]:
            assert cols[e0] // 64 == band
            # a cut happens only at a band boundary or at the chunk size
            if e0 > 0:
                assert cols[e0] // 64 != cols[e0 - 1] // 64 or any(
                    (e0 - s) % chunk == 0 for s in mine[mine[:, 1] < e0][:, 1])
        assert (mine[:-1, 2] >= 4).all() or len(mine) == 1


def test_plan_pieces_independent_of_the_row_range(monkeypatch):
    """A row is cut the same way whichever shard (row range) it falls in: the
    property behind bitwise-identical results across shard counts."""
    monkeypatch.setenv("FMM_BAND_COLS", "64")
    monkeypatch.setenv("FMM_BAND_MINDEG", "64")
    monkeypatch.setenv("FMM_BAND_MINLEN", "4")
    A = _heavy_graph(3)
    _, _, _, whole = _plan_pieces(A)
    key = lambda pc: sorted(map(tuple, pc[:, :3].tolist()))
    parts = []
    for rb, re in ((0, 3000), (3000, 5000), (5000, A.nrows)):
        parts.append(_plan_pieces(A, rb, re)[3])
    assert key(np.concatenate(parts)) == key(whole)


def test_plan_pieces_unsorted_row_keeps_fixed_chunks(monkeypatch):
    monkeypatch.setenv("FMM_BAND_COLS", "64")
    monkeypatch.setenv("FMM_BAND_MINDEG", "64")
    monkeypatch.setenv("FMM_CHUNK", "256")
    A = _heavy_graph(4)
    deg = np.diff(A.row_ptr)
    r = int(np.argmax(deg))
    cols = A.col_idx.copy()
    cols[A.row_ptr[r]:A.row_ptr[r + 1]] = cols[A.row_ptr[r]:A.row_ptr[r + 1]][::-1]
    B = F.CsrMatrix(A.nrows, A.ncols, A.row_ptr, cols, None)
    _, ns, nb, pc = _plan_pieces(B)
    assert nb == ns - 1
    mine = pc[pc[:, 0] == r]
    assert len(mine) == -(-deg[r] // 256) and (np.sort(mine[:, 1]) == np.arange(len(mine)) * 256).all()


def test_wide_threshold_and_bands_depend_on_whole_matrix_only(monkeypatch):
    """fmm_plan_pieces reports the chunk size chosen from the whole matrix's
    nnz, also when asked about a sub-range."""
    A = _heavy_graph(5)
    c_all = _plan_pieces(A)[0]
    assert _plan_pieces(A, 100, 200)[0] == c_all
