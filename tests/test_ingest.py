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
