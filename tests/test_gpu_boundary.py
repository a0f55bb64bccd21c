"""GPU: drop-in boundary semantics (VERDICT r1 "weak" 5, "missing" 2, ADVICE).

* The reference reads A afresh on every fused_mm (kernel.hpp:297-353): a CSR
  whose arrays are edited in place, or rebuilt at the same addresses, must
  give the new result, never one computed from a stale device copy.
* Any d runs (kernel.hpp:192-225 streams d past the blocked limit): d > 1024
  goes to the streamed kernel, checked against the reference-pinned oracle.
* Launches that share a graph's scratch from two streams are ordered.
* Native lifetimes: a context may be destroyed before its graphs.
* Halo masks: fmm_iterate sends only rows a peer reads, bitwise unchanged.
"""
import ctypes as C
import subprocess
import sys
import textwrap

import numpy as np
import pytest

import oracle
from paper_2011_06391_b200 import _lib, configs
from paper_2011_06391_b200 import fusedmm as F
from tests.parity import check_exact, check_tolerance

pytestmark = pytest.mark.gpu


def _rand_graph(seed, m, n, deg, weighted=True):
    rng = np.random.default_rng(seed)
    ent = []
    for r in range(m):
        k = int(rng.integers(0, deg + 1))
        for c in rng.choice(n, size=min(k, n), replace=False):
            ent.append((r, int(c), float(rng.uniform(0.1, 2.0))))
    A = F.csr_from_coo(ent, m, n)
    return A if weighted else F.CsrMatrix(m, n, A.row_ptr, A.col_idx, None)


def test_values_edited_in_place_are_seen():
    A = _rand_graph(1, 300, 300, 12)
    X = F.DenseMatrix(300, 64, np.random.default_rng(2).uniform(-1, 1, 300 * 64))
    spec = F.make_spec(F.App.GCN_FORWARD)
    Z1 = F.fused_mm(A, X, X, spec)
    check_exact(Z1.array, oracle.oracle_fused_mm(A, X, X, spec))
    A.values *= np.float32(3.0)  # same array object, same address
    Z2 = F.fused_mm(A, X, X, spec)
    check_exact(Z2.array, oracle.oracle_fused_mm(A, X, X, spec))
    assert not np.array_equal(Z1.array, Z2.array)


def test_values_assigned_after_unweighted_construction():
    """A built without values, then A.values assigned."""
    A = _rand_graph(3, 200, 200, 10, weighted=False)
    X = F.DenseMatrix(200, 32, np.random.default_rng(4).uniform(-1, 1, 200 * 32))
    spec = F.make_spec(F.App.GCN_FORWARD)
    F.fused_mm(A, X, X, spec)
    A.values = np.random.default_rng(5).uniform(0.5, 2.0, A.nnz()).astype(np.float32)
    check_exact(F.fused_mm(A, X, X, spec).array, oracle.oracle_fused_mm(A, X, X, spec))


def test_columns_edited_in_place_are_seen():
    A = _rand_graph(6, 256, 256, 16)
    X = F.DenseMatrix(256, 128, np.random.default_rng(7).normal(0, 0.1, 256 * 128))
    spec = F.make_spec(F.App.NODE_EMBED_SIGMOID)
    F.fused_mm(A, X, X, spec)
    rng = np.random.default_rng(8)
    for r in range(A.nrows):  # permute each row's columns in place: new storage order
        lo, hi = A.row_ptr[r], A.row_ptr[r + 1]
        A.col_idx[lo:hi] = A.col_idx[lo:hi][rng.permutation(hi - lo)]
    Zg = F.fused_mm(A, X, X, spec)
    check_tolerance(Zg.array, oracle.oracle_fused_mm(A, X, X, spec), A, X, X, spec)


def test_rebuilt_csr_at_same_addresses():
    """A CSR rebuilt in a loop with the same sizes reuses the same buffers:
    emulate that by overwriting every array in place with another graph."""
    A = _rand_graph(9, 400, 400, 8)
    B = _rand_graph(10, 400, 400, 8)
    X = F.DenseMatrix(400, 64, np.random.default_rng(11).uniform(-1, 1, 400 * 64))
    spec = F.make_spec(F.App.GCN_FORWARD)
    F.fused_mm(A, X, X, spec)
    k = min(A.nnz(), B.nnz())
    A.row_ptr[:] = np.minimum(B.row_ptr, k)
    A.col_idx[:k] = B.col_idx[:k]
    A.values[:k] = B.values[:k]
    A.col_idx = A.col_idx[:k]  # a view: same base address
    A.values = A.values[:k]
    check_exact(F.fused_mm(A, X, X, spec).array, oracle.oracle_fused_mm(A, X, X, spec))


@pytest.mark.parametrize("d", [1025, 1500, 2048])
@pytest.mark.parametrize("app", ["sigmoid", "gcn", "fr"])
def test_large_d_streamed_kernel(d, app):
    A = _rand_graph(12 + d, 96, 96, 20, weighted=(app == "gcn"))
    rng = np.random.default_rng(d)
    X = F.DenseMatrix(96, d, rng.normal(0, 0.05, 96 * d))
    spec = {"sigmoid": F.make_spec(F.App.NODE_EMBED_SIGMOID), "gcn": F.make_spec(F.App.GCN_FORWARD),
            "fr": F.make_spec(F.App.FR_LAYOUT, F.AppParams(alpha=0.5))}[app]
    Zg = F.fused_mm(A, X, X, spec)
    Zr = oracle.oracle_fused_mm(A, X, X, spec)
    if app == "gcn":  # vector message, exact scheme: storage-order fold per element
        check_exact(Zg.array, Zr)
    else:
        check_tolerance(Zg.array, Zr, A, X, X, spec)


@pytest.mark.parametrize("spec", [
    F.OpSpec(F.Vop.SUB, F.Rop.SQNORM, F.Sop.TDIST, F.Mop.MUL_VOP, F.Aop.ASUM),
    F.OpSpec(F.Vop.ADD, F.Rop.NOOP, F.Sop.SIGMOID, F.Mop.MUL, F.Aop.AMAX),
    F.OpSpec(F.Vop.MUL, F.Rop.RSUM, F.Sop.SCAL, F.Mop.SEL2ND, F.Aop.AMAX, alpha=0.25),
])
def test_large_d_generic_ops(spec):
    d = 1300
    A = _rand_graph(40, 64, 64, 12)
    rng = np.random.default_rng(41)
    X = F.DenseMatrix(64, d, rng.uniform(-0.05, 0.05, 64 * d))
    Zg = F.fused_mm(A, X, X, spec)
    check_tolerance(Zg.array, oracle.oracle_fused_mm(A, X, X, spec), A, X, X, spec)


def test_large_d_iterate_two_shards_bitwise():
    w = configs.get(3, small=True)
    d = 1100
    X = F.DenseMatrix(w.A.nrows, d, np.random.default_rng(3).uniform(-1, 1, w.A.nrows * d))
    Z1 = F.iterate(w.A, X, w.spec, 2, 1)
    Z2 = F.iterate(w.A, X, w.spec, 2, 2)
    check_exact(Z2.array, Z1.array)


def test_two_streams_share_graph_scratch():
    """FMM_ASYNC launches of one graph on two different streams (set_stream
    between them) are ordered by the library: both results equal the
    synchronous one (split-row partials and fold tickets are shared)."""
    import torch
    w = configs.get(2, small=True)
    dev = torch.device("cuda", 0)
    with F.Context([0]) as ctx:
        g = F.DeviceGraph(ctx, w.A)
        assert g.info().split_rows > 0
        X = torch.from_numpy(w.X.array.copy()).to(dev)
        ref = torch.empty_like(X)
        g.run_device(X.data_ptr(), X.shape[0], X.data_ptr(), ref.data_ptr(), w.d, w.spec,
                     flags=_lib.FMM_DEVICE_PTRS)
        outs = []
        streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
        for k in range(6):
            s = streams[k % 2]
            ctx.set_stream(0, s.cuda_stream)
            Z = torch.empty_like(X)
            g.run_device(X.data_ptr(), X.shape[0], X.data_ptr(), Z.data_ptr(), w.d, w.spec)
            outs.append(Z)
        torch.cuda.synchronize()
        for Z in outs:
            check_exact(Z.cpu().numpy(), ref.cpu().numpy())
        g.free()


def test_context_destroyed_before_graph(tmp_path):
    """fmm_destroy before fmm_graph_free (any finaliser order) is safe; a
    destroyed context rejects further calls."""
    code = textwrap.dedent("""
        import numpy as np
        from paper_2011_06391_b200 import fusedmm as F, _lib
        from paper_2011_06391_b200 import configs
        w = configs.get(1, small=True)
        ctx = F.Context([0])
        g1 = F.DeviceGraph(ctx, w.A)
        g2 = F.DeviceGraph(ctx, w.A)
        ctx.close()          # graphs still alive
        g1.free()
        del g2               # finaliser after the context
        import gc; gc.collect()
        print("LIFETIME_OK")
    """)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    assert r.returncode == 0 and "LIFETIME_OK" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("cfg", [3, 5])
def test_iterate_halo_masks_cut_exchange(cfg):
    """fmm_iterate with 3 shards: only rows another shard reads are stored
    to it; the iterate is bitwise the single-shard one."""
    w = configs.get(cfg, small=True)
    ref = F.iterate(w.A, w.X, w.spec, 3, 1)
    g = F._device_graph(w.A, 3, w.d)
    Z = F.iterate(w.A, w.X, w.spec, 3, 3)
    check_exact(Z.array, ref.array)
    info = g.info()
    assert info.exchange_rows_all == w.A.nrows * 2
    empty = int(np.count_nonzero(np.diff(w.A.row_ptr) == 0))
    # symmetric graph: an empty row has no in-edges, nobody reads it
    assert info.exchange_rows <= info.exchange_rows_all - 2 * empty
    assert info.exchange_rows < info.exchange_rows_all


def test_unaligned_peer_buffer_falls_back_to_masked_shapes():
    """peer buffers that are not 16/32-byte aligned must not be
    stored with vector stores; the call picks the masked shapes and the peer
    receives exactly the rows Z receives."""
    import torch
    w = configs.get(2, small=True)
    dev = torch.device("cuda", 0)
    with F.Context([0]) as ctx:
        g = F.DeviceGraph(ctx, w.A)
        X = torch.from_numpy(w.X.array.copy()).to(dev)
        Z = torch.zeros_like(X)
        peer = torch.zeros(X.numel() + 1, dtype=torch.float32, device=dev)
        g.run_device_peers(X.data_ptr(), X.shape[0], X.data_ptr(), Z.data_ptr(), w.d, w.spec,
                           [peer.data_ptr() + 4], flags=_lib.FMM_DEVICE_PTRS)
        torch.cuda.synchronize()
        check_exact(peer[1:].view(X.shape).cpu().numpy(), Z.cpu().numpy())
        check_tolerance(Z.cpu().numpy(), oracle.oracle_fused_mm(w.A, w.X, w.X, w.spec), w.A, w.X, w.X, w.spec)
        g.free()


def test_concurrent_host_threads_share_the_api():
    """Several host threads calling fused_mm on shared and private graphs:
    every result equals the oracle (the cached graph is never freed under a
    running call: lookup and run hold one lock, the C context a mutex)."""
    import threading
    shared = _rand_graph(50, 200, 200, 10)
    X = F.DenseMatrix(200, 64, np.random.default_rng(51).uniform(-1, 1, 200 * 64))
    spec = F.make_spec(F.App.GCN_FORWARD)
    want_shared = oracle.oracle_fused_mm(shared, X, X, spec)
    errors = []

    def worker(k):
        try:
            own = _rand_graph(60 + k, 200, 200, 6 + k)
            want_own = oracle.oracle_fused_mm(own, X, X, spec)
            for _ in range(8):
                check_exact(F.fused_mm(shared, X, X, spec).array, want_shared)
                check_exact(F.fused_mm(own, X, X, spec).array, want_own)
        except Exception as e:  # noqa: BLE001 - surfaced below
            errors.append(e)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[0]
