"""GPU: every non-USER five-slot combination of ops.hpp:14-18 plus the device
extensions, across the kernel shape families (vectorised lane groups, the
masked scalar-load shapes for ragged d, thread-per-row d <= 4), the golden
vectors produced by the reference itself, and edge cases (empty rows, empty
graph, AMAX identities, weighted / unweighted, Y != X)."""
import itertools
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2011_06391_b200 import fusedmm as F
from tests.parity import check_exact, check_tolerance

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"

VOPS = [F.Vop.ADD, F.Vop.MUL, F.Vop.SEL2ND, F.Vop.SUB]
ROPS = [F.Rop.NOOP, F.Rop.RSUM, F.Rop.RMUL, F.Rop.NORM, F.Rop.SQNORM]
SOPS = [F.Sop.NOOP, F.Sop.SIGMOID, F.Sop.SCAL, F.Sop.TDIST, F.Sop.SQK]
MOPS = [F.Mop.MUL, F.Mop.SEL2ND, F.Mop.MUL_VOP]
AOPS = [F.Aop.ASUM, F.Aop.AMAX]


def random_case(seed, m, n, d, density=0.3, weighted=True, lo=-1.0, hi=1.0):
    rng = np.random.default_rng(seed)
    ent = [(r, c, float(rng.uniform(0.1, 2.0))) for r in range(m) for c in range(n) if rng.random() < density]
    A = F.csr_from_coo(ent, m, n)
    if not weighted:
        A = F.CsrMatrix(m, n, A.row_ptr, A.col_idx, None)
    X = F.DenseMatrix(m, d, rng.uniform(lo, hi, m * d))
    Y = F.DenseMatrix(n, d, rng.uniform(lo, hi, n * d))
    return A, X, Y


def loose_check(Zg, A, X, Y, spec):
    """Semantic check vs the fp64 restatement: per-row error relative to the
    row's scale (catches wrong-op bugs, tolerates reassociation)."""
    Z64 = oracle.oracle_fused_mm(A, X, Y, spec, f64=True)
    Zg = np.asarray(Zg, np.float64)
    fin = np.isfinite(Z64)
    assert np.array_equal(fin, np.isfinite(Zg)), "non-finite pattern differs"
    assert np.array_equal(Zg[~fin], Z64[~fin])
    a = np.where(fin, Zg, 0.0)
    b = np.where(fin, Z64, 0.0)
    scale = np.maximum(np.abs(b).max(axis=1, keepdims=True), 1e-30)
    err = (np.abs(a - b) / scale).max(axis=1)
    # ill-conditioned combinations (e.g. elementwise 1/(1+t) near t = -1) are
    # judged against the fp32 reference's own distance from fp64
    Z32 = np.asarray(oracle.oracle_fused_mm(A, X, Y, spec), np.float64)
    err32 = (np.abs(np.where(fin, Z32, 0.0) - b) / scale).max(axis=1)
    bound = np.maximum(2e-4, 8.0 * err32)
    assert np.all(err <= bound), f"max scaled err {err.max():.3e} (fp32 ref {err32[np.argmax(err)]:.3e})"


COMBOS = [c for c in itertools.product(VOPS, ROPS, SOPS, MOPS, AOPS)
          # RMUL over many elements under/overflows; keep it to small d below
          ]


@pytest.mark.parametrize("d", [3, 16, 128])
def test_all_op_combinations_fast(d):
    A, X, Y = random_case(7 + d, 40, 37, d, weighted=True)
    n_checked = 0
    for (v, r, s, mo, a) in COMBOS:
        if r == F.Rop.RMUL and d > 16:
            continue
        spec = F.OpSpec(v, r, s, mo, a, alpha=0.75, k=1.5)
        Z = F.fused_mm(A, X, Y, spec, 1, opts=F.KernelOptions(exact=False))
        loose_check(Z.array, A, X, Y, spec)
        n_checked += 1
    assert n_checked > 300


@pytest.mark.parametrize("d", [1, 2, 4])
def test_all_op_combinations_exact_thread_per_row(d):
    """d <= 4 runs one thread per row: with FMM_EXACT every reduction is in
    the reference's element order and no FMA is formed, so every combination
    whose scalar op is not the exp-based sigmoid is bit-identical to the
    reference's fused_mm<float> (expf differs by ulps between libm and CUDA)."""
    A, X, Y = random_case(100 + d, 30, 31, d, weighted=True)
    for (v, r, s, mo, a) in COMBOS:
        spec = F.OpSpec(v, r, s, mo, a, alpha=0.75, k=1.5)
        st = F.KernelStats()
        Z = F.fused_mm(A, X, Y, spec, 1, st, opts=F.KernelOptions(exact=True))
        assert st.exact
        Zo = oracle.oracle_fused_mm(A, X, Y, spec)
        if s == F.Sop.SIGMOID:
            loose_check(Z.array, A, X, Y, spec)
        else:
            check_exact(Z.array, Zo)


@pytest.mark.parametrize("path", sorted(GOLDEN.glob("*.npz")), ids=lambda p: p.stem)
def test_golden_vectors_on_device(path):
    from tests.parity import load_golden
    A, X, Y, spec, _lw, Zg = load_golden(path)
    st = F.KernelStats()
    Z = F.fused_mm(A, X, Y, spec, 1, st)
    if st.exact and (F.pattern_of(spec) == F.KnownPattern.SPMM_GCN or X.dim <= 4):
        check_exact(Z.array, Zg)
    else:
        if np.all(np.isfinite(Zg)):
            if np.abs(Zg).max() > 0:
                loose_check(Z.array, A, X, Y, spec)
        else:
            assert np.array_equal(np.isfinite(Z.array), np.isfinite(Zg))


def test_every_make_spec_row_runs_on_device():
    """apps.hpp:22-45: FR_LAYOUT, NODE_EMBED_SIGMOID, GCN_FORWARD and GNN_MLP
    (with the toy MLP hook as the device op Vop.MLP) all run on the GPU."""
    A, X, Y = random_case(77, 60, 60, 32, weighted=True)
    mlp = F.AppParams(alpha=0.5, mlp_vop=F.make_toy_mlp_vop(0.4, 0.6, 0.1))
    for app in (F.App.FR_LAYOUT, F.App.NODE_EMBED_SIGMOID, F.App.GCN_FORWARD, F.App.GNN_MLP):
        spec = F.make_spec(app, mlp)
        assert not spec.has_user_slot()
        Z = F.fused_mm(A, X, Y, spec, 1)
        loose_check(Z.array, A, X, Y, spec)
        if oracle.ref_available():  # the reference itself, through its own toy hook
            Zr = oracle.ref_fused_mm(A, X, Y, spec)
            assert np.max(np.abs(Z.array - Zr)) <= 1e-5 * max(1.0, float(np.abs(Zr).max()))


def test_empty_rows_and_amax_identity():
    A = F.CsrMatrix(4, 4, np.array([0, 0, 2, 2, 3]), np.array([1, 3, 0]))
    X = F.DenseMatrix(4, 8, np.random.default_rng(1).uniform(-1, 1, 32))
    spec = F.OpSpec(F.Vop.MUL, F.Rop.RSUM, F.Sop.SIGMOID, F.Mop.MUL, F.Aop.AMAX)
    for exact in (True, False):
        Z = F.fused_mm(A, X, X, spec, 1, opts=F.KernelOptions(exact=exact))
        assert np.all(Z.array[0] == -np.inf) and np.all(Z.array[2] == -np.inf)
        loose_check(np.where(np.isfinite(Z.array), Z.array, -np.inf), A, X, X, spec)
    Z = F.fused_mm(A, X, X, F.make_spec(F.App.NODE_EMBED_SIGMOID), 1)
    assert not Z.array[0].any() and not Z.array[2].any()


def test_empty_graph_and_zero_rows():
    A = F.CsrMatrix(5, 5)
    X = F.DenseMatrix(5, 16, np.ones(80))
    Z = F.fused_mm(A, X, X, F.make_spec(F.App.NODE_EMBED_SIGMOID), 1)
    assert not Z.array.any()
    A0 = F.CsrMatrix(0, 3)
    Z0 = F.fused_mm(A0, F.DenseMatrix(0, 4), F.DenseMatrix(3, 4), F.make_spec(F.App.GCN_FORWARD), 1)
    assert Z0.array.shape == (0, 4)


def test_y_distinct_from_x_and_rectangular():
    A, X, Y = random_case(5, 50, 70, 64, weighted=True)
    for spec in (F.make_spec(F.App.NODE_EMBED_SIGMOID), F.make_spec(F.App.GCN_FORWARD),
                 F.make_spec(F.App.FR_LAYOUT, F.AppParams(alpha=0.3)), F.tdist_spec()):
        Z = F.fused_mm(A, X, Y, spec, 1)
        Zo = oracle.oracle_fused_mm(A, X, Y, spec)
        if F.pattern_of(spec) == F.KnownPattern.SPMM_GCN:
            check_exact(Z.array, Zo)
        else:
            check_tolerance(Z.array, Zo, A, X, Y, spec)


def test_heavy_rows_split_and_combined():
    """A star + chain graph: hub rows far above the chunk size are split into
    chunks on the fast scheme and folded in chunk order; GCN (exact scheme)
    keeps them whole. Both against the oracle."""
    n = 5000
    ent = [(0, v, 1.0) for v in range(1, n)] + [(v, 0, 1.0) for v in range(1, n)]
    ent += [(1, v, 0.5) for v in range(2, 1500)]
    A = F.csr_from_coo(ent, n, n)
    X = F.DenseMatrix(n, 128, np.random.default_rng(3).normal(0, 0.1, n * 128))
    g = F.DeviceGraph(F.default_context(1), A)
    assert g.info().split_rows == 2
    spec = F.make_spec(F.App.NODE_EMBED_SIGMOID)
    Z = F.fused_mm(A, X, X, spec, 1)
    check_tolerance(Z.array, oracle.oracle_fused_mm(A, X, X, spec), A, X, X, spec)
    gcn = F.make_spec(F.App.GCN_FORWARD)
    check_exact(F.fused_mm(A, X, X, gcn, 1).array, oracle.oracle_fused_mm(A, X, X, gcn))
    # AMAX with splits: max is associative, so the split result is exact
    amax = F.OpSpec(F.Vop.SEL2ND, F.Rop.NOOP, F.Sop.NOOP, F.Mop.MUL, F.Aop.AMAX)
    check_exact(F.fused_mm(A, X, X, amax, 1, opts=F.KernelOptions(exact=False)).array,
                oracle.oracle_fused_mm(A, X, X, amax))


def test_unaligned_device_pointers_use_masked_shapes():
    import ctypes as C
    import torch
    from paper_2011_06391_b200 import _lib
    A, X, _ = random_case(9, 64, 64, 32, weighted=False)
    spec = F.make_spec(F.App.NODE_EMBED_SIGMOID)
    dev = torch.device("cuda", 0)
    buf = torch.zeros(64 * 32 + 1, dtype=torch.float32, device=dev)
    Xd = buf[1:].view(64, 32)  # 4-byte aligned only
    Xd.copy_(torch.from_numpy(X.array))
    Zd = torch.zeros(64 * 32 + 1, dtype=torch.float32, device=dev)[1:].view(64, 32)
    g = F.DeviceGraph(F.Context([0]), A)
    g.run_device(Xd.data_ptr(), 64, Xd.data_ptr(), Zd.data_ptr(), 32, spec,
                 flags=_lib.FMM_DEVICE_PTRS)
    check_tolerance(Zd.cpu().numpy(), oracle.oracle_fused_mm(A, X, X, spec), A, X, X, spec)


def test_cpp_wrapper_runs(tmp_path):
    import subprocess
    from paper_2011_06391_b200 import _lib
    root = Path(__file__).resolve().parents[1]
    exe = tmp_path / "demo"
    r = subprocess.run(["g++", "-std=c++17", f"-I{root/'include'}", str(root / "tests/cpp/wrapper_demo.cpp"),
                        f"-L{_lib.LIB_PATH.parent}", "-lfusedmm_cuda", f"-Wl,-rpath,{_lib.LIB_PATH.parent}",
                        "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "wrapper ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("k", [1.0, 0.25, 4.0, -2.0, 2.0 ** -120, 2.0 ** 120, 3.0, 0.1])
def test_sqk_division_bit_exact_for_every_k(k):
    """SOP_SQK divides by k; for k a power of two the kernels multiply by the
    exact reciprocal instead (the same correctly rounded value). Bit-exact
    against the reference order on the exact scheme for powers of two,
    extreme exponents (reciprocal near the normal range limits) and
    non-powers (IEEE division kept)."""
    A, X, Y = random_case(int(abs(np.log2(abs(k)))) + 5, 50, 50, 2, weighted=False, lo=-3.0, hi=3.0)
    spec = F.fr_attract_spec(k)
    Z = F.fused_mm(A, X, Y, spec, 1, opts=F.KernelOptions(exact=True))
    check_exact(Z.array, oracle.oracle_fused_mm(A, X, Y, spec))


def test_tune_lane_width_and_variant_option():
    """tune_lane_width (kernel.hpp:382-402) times the device shape variants
    and returns one; every variant gives the same result within the fast
    scheme's tolerance (bitwise across runs of one variant)."""
    A, X, Y = random_case(77, 300, 300, 128, density=0.05, weighted=False)
    spec = F.make_spec(F.App.NODE_EMBED_SIGMOID)
    lw = F.tune_lane_width(A, X, Y, spec, 1, repeats=1)
    assert lw in (4, 8, 16)  # the reference's contract
    Zl = F.fused_mm(A, X, Y, spec, 1, opts=F.KernelOptions(lane_width=lw))
    check_tolerance(Zl.array, oracle.oracle_fused_mm(A, X, Y, spec), A, X, Y, spec)
    v = F.tune_variant(A, X, Y, spec, 1, repeats=1)
    assert v in F.SHAPE_VARIANTS
    Z0 = F.fused_mm(A, X, Y, spec, 1, opts=F.KernelOptions(variant=v))
    Z1 = F.fused_mm(A, X, Y, spec, 1, opts=F.KernelOptions(variant=v))
    assert np.array_equal(Z0.array, Z1.array)
    Zo = oracle.oracle_fused_mm(A, X, Y, spec)
    for var in (-1, 20, 21):
        Zv = F.fused_mm(A, X, Y, spec, 1, opts=F.KernelOptions(variant=var))
        check_tolerance(Zv.array, Zo, A, X, Y, spec)
