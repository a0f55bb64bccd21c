"""GPU: the one-process-per-GPU sharding path (shard.py, bench.py under
torchrun) on a one-GPU box. Ranks share GPU 0 and talk over gloo: nothing
waits on another rank inside a kernel (the exchange is host-driven
broadcasts), so this exercises the real device compute, the part1d row
blocks and the slice exchange without needing 2 GPUs. Timings are not
meaningful here."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, iters, out, exchange="broadcast"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2011_06391_b200 import configs
        from paper_2011_06391_b200.shard import ShardedFusedMM
        w = configs.get(cfg, small=True)
        # explicit lifetime: graph and context are released here, not by
        # finalisers during interpreter shutdown
        with ShardedFusedMM(w.A, w.d, w.spec, device=torch.device("cuda", 0), exchange=exchange) as sh:
            X0 = torch.from_numpy(w.X.array.copy()).cuda()
            Z = sh.iterate(X0, iters)
            torch.cuda.synchronize()
            if rank == 0:
                np.save(out, Z.cpu().numpy())
            if exchange == "fused":
                # halo masks: rows no peer reads are never sent
                assert sh.exchange_rows < sh.exchange_rows_all, (sh.exchange_rows, sh.exchange_rows_all)
            del X0, Z
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["broadcast", "fused"])
@pytest.mark.parametrize("cfg,iters,world", [(3, 3, 2), (2, 2, 2), (3, 4, 3)])
def test_sharded_device_iterate_ranks(tmp_path, cfg, iters, world, exchange):
    """fused: the kernels of every rank store their z rows into the other
    ranks' next-X buffers (CUDA IPC mappings, fmm_run_peers); broadcast:
    post-kernel slice broadcasts. Both bitwise equal to one process."""
    from paper_2011_06391_b200 import configs
    from paper_2011_06391_b200 import fusedmm as F
    from tests.parity import check_exact
    out = str(tmp_path / "z.npy")
    mp.start_processes(_worker, args=(world, _free_port(), cfg, iters, out, exchange), nprocs=world, join=True,
                       start_method="spawn")
    w = configs.get(cfg, small=True)
    ref = F.iterate(w.A, w.X, w.spec, iters, 1)
    check_exact(np.load(out), ref.array)


@pytest.mark.parametrize("config", [2, 3])
def test_bench_torchrun_two_ranks_shared_gpu(config):
    """bench.py under torchrun: config 2 (one call, Z row-sharded) and config
    3 (iterative: the step carries the halo exchange, fused into the kernel)."""
    env = dict(os.environ, FMM_BENCH_SHARE_GPU="1", FMM_GEN="device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--config", str(config)]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["value"] > 0 and rec["gpu_launches"] > 0
    ex = rec["exchange"]
    if config == 3:
        assert ex["in_step"] and ex["cut_by_masks"] > 0.38
        assert ex["bytes_per_step_total"] < ex["bytes_per_step_without_halo_masks"]
    else:
        assert not ex["in_step"] and ex["halo_bytes_per_iteration_if_iterated"] > 0
