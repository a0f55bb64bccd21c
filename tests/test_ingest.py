"""Device-side graph construction: fmm_csr_from_coo
against the reference's csr_from_coo (matrix.hpp:87-140) and its CPU
restatement, the R-MAT generator (rmat.hpp:24-61 = insertion stream ->
csr_from_coo) built on the device against the reference's rmat_generate, and
fmm_csr_sym_unique against the host builder of the BASELINE graphs.
CPU tests pin the restatement; GPU tests are bit-exact parity."""
import numpy as np
import pytest

import oracle
from paper_2011_06391_b200 import configs
from paper_2011_06391_b200 import fusedmm as F

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def coo_case(seed, m, n, cnt, dup_frac=0.5):
    rng = np.random.default_rng(seed)
    r = rng.integers(0, max(m, 1), cnt)
    c = rng.integers(0, max(n, 1), cnt)
    k = int(cnt * dup_frac)
    if cnt and k:  # force repeats of earlier (row, col) pairs
        src = rng.integers(0, cnt, k)
        dst = rng.integers(0, cnt, k)
        r[dst] = r[src]
        c[dst] = c[src]
    v = rng.uniform(0.1, 2.0, cnt).astype(np.float32)
    return r, c, v


def same_csr(a, b):
    (rp1, c1, v1), (rp2, c2, v2) = a, b
    assert np.array_equal(rp1, rp2)
    assert np.array_equal(c1, c2)
    if v1 is not None and v2 is not None:
        assert np.array_equal(np.asarray(v1, np.float32).view(np.uint32), np.asarray(v2, np.float32).view(np.uint32))


@needs_ref
@pytest.mark.parametrize("seed,m,n,cnt", [(0, 50, 40, 600), (1, 1, 1, 30), (2, 300, 7, 2000), (3, 9, 900, 50),
                                          (4, 5, 5, 0), (5, 1000, 1000, 5000)])
def test_oracle_csr_from_coo_matches_reference(seed, m, n, cnt):
    r, c, v = coo_case(seed, m, n, cnt)
    same_csr(oracle.oracle_csr_from_coo(r, c, v, m, n), oracle.ref_csr_from_coo(r, c, v, m, n))


@needs_ref
def test_oracle_csr_from_coo_out_of_bounds_raises_like_reference():
    for rows, cols in (([0, 3], [0, 0]), ([0, -1], [0, 0]), ([0, 0], [0, 4])):
        with pytest.raises(ValueError):
            oracle.ref_csr_from_coo(rows, cols, None, 3, 4)
        with pytest.raises(ValueError):
            oracle.oracle_csr_from_coo(rows, cols, None, 3, 4)


@needs_ref
def test_rmat_stream_through_oracle_csr_from_coo_is_rmat_generate():
    rows, cols = configs.rmat_stream(10, 8, 3)
    rp, cl, vl = oracle.ref_rmat(10, 8, 3)
    same_csr(oracle.oracle_csr_from_coo(rows, cols, None, 1 << 10, 1 << 10), (rp, cl, vl))


# ---------------------------------------------------------------- device
@pytest.mark.gpu
@pytest.mark.parametrize("seed,m,n,cnt", [(0, 50, 40, 600), (1, 1, 1, 30), (2, 300, 7, 2000), (3, 9, 900, 50),
                                          (4, 5, 5, 0), (5, 1000, 1000, 5000), (6, 70000, 3, 200000),
                                          (7, 3, 100000, 100000)])
def test_device_csr_from_coo_bit_exact(seed, m, n, cnt):
    r, c, v = coo_case(seed, m, n, cnt)
    A = F.csr_from_coo_device(r, c, v, m, n)
    want = oracle.ref_csr_from_coo(r, c, v, m, n) if oracle.ref_available() else oracle.oracle_csr_from_coo(r, c, v, m, n)
    same_csr((A.row_ptr, A.col_idx, A.values), want)
    assert F.validate(A) is None


@pytest.mark.gpu
def test_device_csr_from_coo_unweighted_and_errors():
    r, c, _ = coo_case(11, 40, 40, 500)
    A = F.csr_from_coo_device(r, c, None, 40, 40)
    same_csr((A.row_ptr, A.col_idx, A.values), oracle.oracle_csr_from_coo(r, c, None, 40, 40))
    for rows, cols in (([0, 3], [0, 0]), ([0, -1], [0, 0]), ([0, 0], [0, 4])):
        with pytest.raises(F.InvalidArgument):
            F.csr_from_coo_device(rows, cols, None, 3, 4)


@pytest.mark.gpu
@pytest.mark.parametrize("scale,ef,seed", [(10, 8, 3), (14, 16, 1)])
def test_device_rmat_generate_matches_reference(scale, ef, seed):
    """rmat_generate = the insertion stream folded by csr_from_coo; the
    device fold equals the reference generator bitwise (self-loops kept,
    duplicates summed into values > 1)."""
    rows, cols = configs.rmat_stream(scale, ef, seed)
    A = F.csr_from_coo_device(rows, cols, None, 1 << scale, 1 << scale)
    if oracle.ref_available():
        want = oracle.ref_rmat(scale, ef, seed)
    else:
        want = oracle.oracle_csr_from_coo(rows, cols, None, 1 << scale, 1 << scale)
    same_csr((A.row_ptr, A.col_idx, A.values), want)
    assert A.values.max() > 1.0  # duplicates were summed


@pytest.mark.gpu
@pytest.mark.parametrize("scale,ef,seed", [(12, 16, 1), (20, 16, 1)])
def test_device_sym_unique_matches_host_builder(scale, ef, seed):
    """The BASELINE graph recipe (configs 2/3/5) built on the device equals
    the host builder (and so the survey's probe figures at scale 20)."""
    rows, cols = configs.rmat_stream(scale, ef, seed)
    A = F.csr_sym_unique_device(rows, cols, 1 << scale)
    H = configs.rmat_sym(scale, ef, seed)
    assert np.array_equal(A.row_ptr, H.row_ptr)
    assert np.array_equal(A.col_idx, H.col_idx)
    if scale == 20:
        assert A.nnz() == 31_398_704


@pytest.mark.gpu
def test_device_sym_unique_edge_cases():
    A = F.csr_sym_unique_device([0, 1, 1, 2], [0, 2, 2, 1], 3)  # self-loop dropped, duplicates merged
    assert A.row_ptr.tolist() == [0, 0, 1, 2] and A.col_idx.tolist() == [2, 1]
    B = F.csr_sym_unique_device([0, 1], [0, 2], 3, drop_self=False, symmetrize=False)
    assert B.row_ptr.tolist() == [0, 1, 2, 2] and B.col_idx.tolist() == [0, 2]
    E = F.csr_sym_unique_device([], [], 4)
    assert E.row_ptr.tolist() == [0] * 5 and E.nnz() == 0
    with pytest.raises(F.InvalidArgument):
        F.csr_sym_unique_device([0], [9], 4)


# ------------------------------------------------------------ MatrixMarket
MM_CASES = {
    "general_real": "%%MatrixMarket matrix coordinate real general\n% comment\n\n3 4 5\n1 2 0.5\n3 4 -1.25e-3\n1 2 2.0\n2 1 7\n3 3 1e10\n",
    "symmetric_pattern": "%%MatrixMarket matrix coordinate pattern symmetric\n4 4 4\n2 1\n3 1\n4 4\n3 1\n",
    "integer": "%%MatrixMarket matrix coordinate integer general\n2 2 2\n1 1 3\n2 2 -4\n",
    "empty": "%%MatrixMarket matrix coordinate real general\n5 5 0\n",
    # stream-extraction corner cases the reference accepts
    "crlf": "%%MatrixMarket matrix coordinate real general\r\n2 3 2\r\n1 3 0.5\r\n2 1 -2\r\n",
    "signs_tabs": "%%MatrixMarket  matrix\tcoordinate real general extra\n2 2 2\n+1\t+2 +2.5\n2 2 -.5\n",
    "value_prefixes": "%%MatrixMarket matrix coordinate real general\n3 3 4\n1 1 1.5abc\n2 2 0x1p3\n3 3 5.\n1 3 1e-310\n",
    "no_final_newline": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n2 1",
}
MM_BAD = {
    "header": "%%MatrixMarket matrix array real general\n2 2 0\n",
    "field": "%%MatrixMarket matrix coordinate complex general\n2 2 0\n",
    "symmetry": "%%MatrixMarket matrix coordinate real hermitian\n2 2 0\n",
    "size": "%%MatrixMarket matrix coordinate real general\n2 x 0\n",
    "dims": "%%MatrixMarket matrix coordinate real general\n0 2 0\n",
    "entry": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1\n",
    "value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 abc\n",
    "bounds": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "count": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
    "empty_file": "",
    # stream-extraction corner cases the reference rejects
    "inf_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 inf\n",
    "nan_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 nan\n",
    "exp_no_digits": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1e\n",
    "exp_overflow": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 -1e999\n",
    "dot_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 .\n",
    "int_overflow": "%%MatrixMarket matrix coordinate real general\n2 2 1\n99999999999999999999 1 1.0\n",
    "float_index": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1.0 1 1.0\n",
    "spaced_comment": "%%MatrixMarket matrix coordinate real general\n2 2 1\n % not a comment\n1 1 1\n",
    "crlf_blank": "%%MatrixMarket matrix coordinate real general\r\n\r\n2 2 0\r\n",
    "header_short": "%%MatrixMarket matrix coordinate\n2 2 0\n",
    "header_case": "%%matrixmarket matrix coordinate real general\n2 2 0\n",
    "size_missing": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "size_float": "%%MatrixMarket matrix coordinate real general\n2.0 2 1\n",
    "neg_dims": "%%MatrixMarket matrix coordinate real general\n2 -1 0\n",
    "count_no_newline": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 2",
    "count_over": "%%MatrixMarket matrix coordinate pattern symmetric\n2 2 1\n1 2\n2 1\n",
}


@needs_ref
@pytest.mark.parametrize("name", sorted(MM_BAD))
def test_matrix_market_errors_match_reference(tmp_path, name):
    """Parse errors are detected on the host before any device work, with
    the reference's MmParseError text."""
    path = tmp_path / f"{name}.mtx"
    path.write_text(MM_BAD[name])
    with pytest.raises(ValueError) as want:
        oracle.ref_read_matrix_market(path)
    with pytest.raises(F.MmParseError) as got:
        F.read_matrix_market(path)
    assert str(got.value) == str(want.value)


@needs_ref
def test_write_matrix_market_matches_reference_bytes(tmp_path):
    rng = np.random.default_rng(3)
    r, c, v = coo_case(3, 30, 20, 200)
    rp, cl, vl = oracle.ref_csr_from_coo(r, c, v * np.float32(1e-3) - 0.1, 30, 20)
    A = F.CsrMatrix(30, 20, rp, cl, vl)
    F.write_matrix_market(A, tmp_path / "ours.mtx")
    oracle.ref_write_matrix_market(tmp_path / "ref.mtx", 30, 20, rp, cl, vl)
    assert (tmp_path / "ours.mtx").read_bytes() == (tmp_path / "ref.mtx").read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(MM_CASES))
def test_device_read_matrix_market_matches_reference(tmp_path, name):
    path = tmp_path / f"{name}.mtx"
    path.write_text(MM_CASES[name])
    A = F.read_matrix_market(path)
    if oracle.ref_available():
        m, n, rp, cl, vl = oracle.ref_read_matrix_market(path)
        assert (A.nrows, A.ncols) == (m, n)
        same_csr((A.row_ptr, A.col_idx, A.values), (rp, cl, vl))
    assert F.validate(A) is None


@pytest.mark.gpu
def test_matrix_market_round_trip(tmp_path):
    """write -> read is the identity on a CSR with unique columns (values
    printed with 17 significant digits round-trip float32 exactly)."""
    r, c, v = coo_case(21, 300, 250, 4000)
    A = F.csr_from_coo_device(r, c, v, 300, 250)
    F.write_matrix_market(A, tmp_path / "a.mtx")
    B = F.read_matrix_market(tmp_path / "a.mtx")
    same_csr((A.row_ptr, A.col_idx, A.values), (B.row_ptr, B.col_idx, B.values))


# ---------------------------------------- the reference's own IO tests, ported
def _mm(tmp_path, name, body):
    path = tmp_path / name
    path.write_text(body)
    return path


@pytest.mark.gpu
def test_ref_io_pattern_symmetric_expands_to_2_cycle(tmp_path):
    """test_io.cpp:33-43"""
    A = F.read_matrix_market(_mm(tmp_path, "s.mtx", "%%MatrixMarket matrix coordinate pattern symmetric\n2 2 1\n2 1\n"))
    assert A.nnz() == 2 and A.row_ptr.tolist() == [0, 1, 2] and A.values.tolist() == [1.0, 1.0]


@pytest.mark.gpu
def test_ref_io_real_general_preserves_weights(tmp_path):
    """test_io.cpp:45-55"""
    A = F.read_matrix_market(_mm(tmp_path, "r.mtx", "%%MatrixMarket matrix coordinate real general\n"
                                 "% a comment\n2 2 2\n1 2 2.5\n2 1 -1.25\n"))
    assert A.values.tolist() == [2.5, -1.25]


def test_ref_io_errors_report_line_and_reject(tmp_path):
    """test_io.cpp:57-85 (parse errors are raised on the host, no GPU)"""
    with pytest.raises(F.MmParseError) as e:
        F.read_matrix_market(_mm(tmp_path, "o.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n"))
    assert ":3:" in str(e.value)
    with pytest.raises(F.MmParseError):
        F.read_matrix_market(_mm(tmp_path, "h.mtx", "%%NotMatrixMarket nope\n1 1 0\n"))
    with pytest.raises(F.MmParseError):
        F.read_matrix_market(_mm(tmp_path, "v.mtx", "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 abc\n"))


@pytest.mark.gpu
def test_ref_io_write_read_round_trips_generated_graph(tmp_path):
    """test_io.cpp:87-101: rmat_generate (scale 7, ef 4, seed 99) on the
    device, written and read back unchanged."""
    A = configs.rmat_generate(7, 4, 99)
    F.write_matrix_market(A, tmp_path / "rt.mtx")
    B = F.read_matrix_market(tmp_path / "rt.mtx")
    assert A.nrows == B.nrows
    same_csr((A.row_ptr, A.col_idx, A.values), (B.row_ptr, B.col_idx, B.values))


@pytest.mark.gpu
def test_ref_io_rmat_size_contract_and_determinism():
    """test_io.cpp:103-118"""
    A = configs.rmat_generate(10, 8, 5)
    assert A.nrows == 1024 and 0 < A.nnz() <= 8192 and F.validate(A) is None
    B = configs.rmat_generate(10, 8, 5)
    same_csr((A.row_ptr, A.col_idx, A.values), (B.row_ptr, B.col_idx, B.values))


# ------------------------------------------- device R-MAT (jump-ahead MT64)
def _mt64_outputs_from_window(w: np.ndarray, count: int) -> np.ndarray:
    """Next `count` outputs of the word recurrence from a 312-word window
    (numpy restatement of the twist + tempering, test-side)."""
    A, UM, LM = np.uint64(0xB5026F5AA96619E9), np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)
    out = []
    x = w.astype(np.uint64).copy()
    while sum(o.size for o in out) < count:
        nw = np.zeros(312, np.uint64)

        def nxt(x0, x1, xm):
            y = (x0 & UM) | (x1 & LM)
            return xm ^ (y >> np.uint64(1)) ^ np.where((x1 & np.uint64(1)) != 0, A, np.uint64(0))
        nw[:156] = nxt(x[:156], x[1:157], x[156:312])
        nw[156:311] = nxt(x[156:311], x[157:312], nw[0:155])
        nw[311] = nxt(x[311:312], nw[0:1], nw[155:156])[0]
        y = nw.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        out.append(y)
        x = nw
    return np.concatenate(out)[:count]


@needs_ref
@pytest.mark.parametrize("seed,pos", [(1, 0), (1, 1), (4, 311), (4, 312), (2, 123457), (7, 10 ** 9 + 7),
                                      (1, 24 * 32 * (1 << 24) - 624)])
def test_mt64_jump_ahead_equals_std_mt19937_64(seed, pos):
    """fmm_mt64_window(seed, p): the polynomial jump-ahead gives the window
    whose next outputs are std::mt19937_64(seed) outputs p, p+1, ... — up to
    config 5's last sub-stream (scale 24 x 32 edges x 24 words)."""
    import ctypes as C
    from paper_2011_06391_b200 import _lib
    w = np.zeros(312, np.uint64)
    assert _lib.lib().fmm_mt64_window(seed, pos, w.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
    want = np.zeros(700, np.uint64)
    L = oracle.ref_lib()
    L.fmm_ref_mt64_outputs.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.POINTER(C.c_uint64)]
    L.fmm_ref_mt64_outputs(seed, pos, want.size, want.ctypes.data_as(C.POINTER(C.c_uint64)))
    assert np.array_equal(_mt64_outputs_from_window(w, want.size), want)


@pytest.mark.gpu
@pytest.mark.parametrize("scale,ef,seed", [(10, 16, 1), (13, 8, 2), (12, 32, 4), (7, 3, 9)])
def test_device_rmat_stream_equals_host_stream(scale, ef, seed):
    """The raw insertion stream generated on the device (jump-ahead
    sub-streams) equals the sequential host stream (pinned to the
    reference's rmat_generate by test_oracle.py)."""
    r_d, c_d = configs.rmat_device(scale, ef, seed, recipe=2)
    r_h, c_h = configs.rmat_stream(scale, ef, seed)
    assert np.array_equal(r_d, r_h) and np.array_equal(c_d, c_h)


@pytest.mark.gpu
@pytest.mark.parametrize("scale,ef,seed", [(9, 16, 1), (12, 8, 5)])
def test_device_rmat_generate_recipe_equals_reference(scale, ef, seed):
    A = configs.rmat_device(scale, ef, seed, recipe=0)
    if oracle.ref_available():
        same_csr((A.row_ptr, A.col_idx, A.values), oracle.ref_rmat(scale, ef, seed))


@pytest.mark.gpu
@pytest.mark.parametrize("scale,ef,seed", [(13, 16, 1), (20, 16, 1)])
def test_device_rmat_baseline_recipe_equals_host_builder(scale, ef, seed):
    """The BASELINE graph built wholly on the device equals the host builder
    (config 2 at its full size included)."""
    A = configs.rmat_device(scale, ef, seed, recipe=1)
    B = configs.rmat_sym(scale, ef, seed)
    assert np.array_equal(A.row_ptr, B.row_ptr) and np.array_equal(A.col_idx, B.col_idx)
