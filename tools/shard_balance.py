"""Per-shard kernel time of the part1d row blocks, measured one shard at a
time on one B200 (tool; JSON lines). With one GPU reachable, this is the
compute side of multi-GPU scaling: at G GPUs each GPU runs exactly its shard's
kernel, so max over shards / (one-shard time) bounds the compute speed-up,
and the exchange volume per iteration is reported beside it.

    python tools/shard_balance.py --config 2 [--gpus 1,2,4,8] [--halo]

--halo: each shard's kernel also performs its halo exchange stores (the
z rows its peers read, per-row peer masks) into G-1 local stand-in peer
buffers — the kernel-side cost of the fused exchange, with local HBM in
place of NVLink.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--gpus", default="1,2,4,8")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--partition", default="both", choices=("part1d", "weighted", "both"))
    ap.add_argument("--halo", action="store_true")
    a = ap.parse_args()
    import torch
    from paper_2011_06391_b200 import configs
    from paper_2011_06391_b200 import fusedmm as F

    w = configs.get(a.config)
    A, spec, d = w.A, w.spec, w.d
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    X = torch.from_numpy(w.X.array).to(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    ctx = F.Context([0])
    ctx.set_stream(0, stream.cuda_stream)
    parts = ["part1d", "weighted"] if a.partition == "both" else [a.partition]
    base = None
    for part, G in [(pt, int(x)) for pt in parts for x in a.gpus.split(",")]:
        b = F.part1d(A, G).boundaries if part == "part1d" else F.shard_bounds(A, G, d).boundaries
        times, nnzs = [], []
        need = None
        if a.halo and G > 1:  # every shard's column-use bitmap (the rows it reads)
            need = []
            for q in range(G):
                gq = F.DeviceGraph(ctx, A, b[q], b[q + 1])
                need.append(gq.column_use())
                gq.free()
        sent_rows = []
        for s in range(G):
            rb, re = b[s], b[s + 1]
            g = F.DeviceGraph(ctx, A, rb, re)
            Z = torch.empty((max(re - rb, 1), d), dtype=torch.float32, device=dev)
            peers = []
            if need is not None:
                mask = np.zeros(re - rb, np.uint8)
                slot = 0
                for q in range(G):
                    if q != s:
                        mask |= (need[q][rb:re] != 0).astype(np.uint8) << slot
                        slot += 1
                g.set_peer_mask(mask, G - 1)
                sent_rows.append(int(g.info().exchange_rows))
                peers = [torch.empty((max(re - rb, 1), d), dtype=torch.float32, device=dev) for _ in range(G - 1)]

            def call():
                if peers:
                    g.run_device_peers(X.data_ptr(), A.nrows, X.data_ptr(), Z.data_ptr(), d, spec,
                                       [pb.data_ptr() for pb in peers])
                else:
                    g.run_device(X.data_ptr(), A.nrows, X.data_ptr(), Z.data_ptr(), d, spec)
            call()
            ts = []
            for _ in range(a.iters):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                call()
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            del peers
            times.append(float(np.median(ts)))
            nnzs.append(int(A.row_ptr[re] - A.row_ptr[rb]))
            g.free()
            del Z
        tmax = max(times)
        if base is None:
            base = tmax
        # per iteration every GPU receives the other shards' Z rows
        recv_bytes = int(A.nrows * d * 4 * (G - 1) / G)
        print(json.dumps({"config": a.config, "partition": part, "gpus": G, "shard_ms": [round(t, 4) for t in times],
                          "shard_nnz": nnzs, "max_ms": tmax, "mean_ms": float(np.mean(times)),
                          "imbalance_max_over_mean": tmax / float(np.mean(times)),
                          "compute_speedup_vs_1": base / tmax,
                          "exchange_bytes_received_per_gpu_per_iteration": recv_bytes,
                          "halo_stores": bool(need is not None),
                          "halo_bytes_sent_per_shard": [r * d * 4 for r in sent_rows]}), flush=True)


if __name__ == "__main__":
    main()
