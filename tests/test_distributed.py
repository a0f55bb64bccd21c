"""CPU, world_size 2 over gloo: the multi-GPU row-sharding layer
(paper_2011_06391_b200/shard.py) — part1d row blocks, per-rank slices, the
per-iteration slice exchange — with the per-shard compute injected (the CPU
oracle stands in for the device kernel here; on GPUs it is libfusedmm_cuda).
The result must be bitwise identical to the single-process run, as the
reference demands across worker counts (kernel.hpp:290-295)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_compute(A, spec):
    import oracle
    from paper_2011_06391_b200 import fusedmm as F

    def compute(X, Y, rb, re):
        Xm = F.DenseMatrix.wrap(X.numpy())
        Ym = Xm if Y is X else F.DenseMatrix.wrap(Y.numpy())
        Z = oracle.oracle_fused_mm(A, Xm, Ym, spec, rows=np.arange(rb, re), threads=1)
        return torch.from_numpy(Z)
    return compute


def _worker(rank, world, port, cfg, iters, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2011_06391_b200 import configs
        from paper_2011_06391_b200.shard import ShardedFusedMM
        w = configs.get(cfg, small=True)
        sh = ShardedFusedMM(w.A, w.d, w.spec, compute=_oracle_compute(w.A, w.spec))
        X0 = torch.from_numpy(w.X.array.copy())
        Z = sh.iterate(X0, iters)
        one = sh.step(X0)
        if rank == 0:
            np.savez(out_path, Z=Z.numpy(), bounds=np.array(sh.bounds))
        np.save(f"{out_path}.step{rank}.npy", one.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,iters", [(3, 3), (5, 2), (2, 1)])
def test_two_rank_iterate_bitwise_equals_single(tmp_path, cfg, iters):
    import oracle
    from paper_2011_06391_b200 import configs
    from paper_2011_06391_b200 import fusedmm as F

    out = str(tmp_path / "res.npz")
    mp.start_processes(_worker, args=(2, _free_port(), cfg, iters, out), nprocs=2, join=True,
                       start_method="spawn")
    res = np.load(out)
    w = configs.get(cfg, small=True)
    X = w.X
    for _ in range(iters):
        X = F.DenseMatrix.wrap(oracle.oracle_fused_mm(w.A, X, X, w.spec))
    assert np.array_equal(res["Z"].view(np.uint32), X.array.view(np.uint32))
    b = res["bounds"].tolist()
    assert b == F.shard_bounds(w.A, 2, w.d).boundaries
    # each rank's one-step slice is its row block of the full result
    Z1 = oracle.oracle_fused_mm(w.A, w.X, w.X, w.spec)
    for r in range(2):
        s = np.load(f"{out}.step{r}.npy")
        assert np.array_equal(s, Z1[b[r]:b[r + 1]])
