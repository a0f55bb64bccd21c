"""Kernel-shape sweep (tuning tool, GPU): for a config, time every shape
variant of the fused kernel with CUDA events (L2 flushed between launches)
and check each against the oracle on sampled rows.

    python tests/sweep_variants.py --config 2 --variants -1,0,1,2,3,4
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--variants", default="-1,0,1,2,3,4")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--env", default="", help="NAME=v1,v2,...: sweep an environment variable too")
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--hot", type=int, default=0,
                    help="characterisation: remap every column to col %% HOT (an L2-resident gather set)")
    ap.add_argument("--hot-min-deg", type=int, default=0,
                    help="with --hot: remap only the columns of rows with at least this many edges")
    a = ap.parse_args()

    import torch
    import oracle
    from paper_2011_06391_b200 import configs, _lib
    from paper_2011_06391_b200 import fusedmm as F
    from tests.parity import check_tolerance, check_exact

    w = configs.get(a.config, small=a.small)
    A, X, spec, d = w.A, w.X, w.spec, w.d
    if a.hot:
        from paper_2011_06391_b200.fusedmm import CsrMatrix
        cols = A.col_idx % a.hot
        if a.hot_min_deg > 0:
            heavy = np.repeat(np.diff(A.row_ptr) >= a.hot_min_deg, np.diff(A.row_ptr))
            cols = np.where(heavy, cols, A.col_idx)
        A = CsrMatrix(A.nrows, A.ncols, A.row_ptr, cols, A.values)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    Xd = torch.from_numpy(X.array).to(dev)
    Zd = torch.empty_like(Xd)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    deg = np.diff(A.row_ptr)
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([np.argsort(-deg)[:16], rng.integers(0, A.nrows, 2048)]))
    Zo = oracle.oracle_fused_mm(A, X, X, spec, rows=rows)
    nnzd = A.nnz() * d
    flags = _lib.FMM_DEVICE_PTRS | _lib.FMM_ASYNC | (_lib.FMM_EXACT if a.exact else 0)
    out = []
    env_name, env_vals = (a.env.split("=", 1)[0], a.env.split("=", 1)[1].split(",")) if a.env else ("", [""])
    for v, ev in [(int(s), e) for s in a.variants.split(",") for e in env_vals]:
        os.environ["FMM_VARIANT"] = str(v)
        if env_name:
            os.environ[env_name] = ev
        ctx = F.Context([0])
        ctx.set_stream(0, stream.cuda_stream)
        g = F.DeviceGraph(ctx, A)
        run = lambda: g.run_device(Xd.data_ptr(), A.nrows, Xd.data_ptr(), Zd.data_ptr(), d, spec, flags=flags)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        times = []
        for _ in range(a.iters):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        Zs = Zd.cpu().numpy()[rows]
        if w.exact or a.exact:
            try:
                check_exact(Zs, Zo)
                par = "bit-exact"
            except AssertionError as e:
                par = f"NOT EXACT: {e}"
        else:
            try:
                par = f"max_row_err {check_tolerance(Zs, Zo, A, X, X, spec, rows=rows)['max_row_err']:.2e}"
            except AssertionError as e:
                par = f"FAIL {e}"
        ms = float(np.median(times))
        rec = {"config": a.config, "variant": v, "env": f"{env_name}={ev}" if env_name else "", "median_ms": ms, "min_ms": float(min(times)),
               "nnzd_per_s": nnzd / (ms / 1e3), "alg_GBps": w.alg_bytes() / (ms / 1e3) / 1e9, "parity": par}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        del g, ctx
    return 0


if __name__ == "__main__":
    sys.exit(main())
