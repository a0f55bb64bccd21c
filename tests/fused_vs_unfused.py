"""Fused vs unfused on the B200 (tool; JSON lines): the paper's claim
(the reference's bench.hpp:114-125 comparison) measured on
the device — time and the materialised message bytes of the unfused
SDDMM -> SpMM pipeline against the single fused pass.

    python tests/fused_vs_unfused.py --configs 1,2
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
    ap.add_argument("--configs", default="1,2")
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    import torch
    from paper_2011_06391_b200 import configs, _lib
    from paper_2011_06391_b200 import fusedmm as F

    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for c in [int(x) for x in a.configs.split(",")]:
        w = configs.get(c)
        ctx = F.Context([0])
        ctx.set_stream(0, stream.cuda_stream)
        g = F.DeviceGraph(ctx, w.A)
        X = torch.from_numpy(w.X.array).to(dev)
        Z = torch.empty_like(X)
        m, d = w.A.nrows, w.d
        fused = lambda: g.run_device(X.data_ptr(), m, X.data_ptr(), Z.data_ptr(), d, w.spec,  # noqa: E731
                                     flags=_lib.FMM_DEVICE_PTRS | _lib.FMM_ASYNC | _lib.FMM_FAST)
        unfused = lambda: g.run_unfused_device(X.data_ptr(), m, X.data_ptr(), Z.data_ptr(), d, w.spec,  # noqa: E731
                                               flags=_lib.FMM_DEVICE_PTRS | _lib.FMM_ASYNC)
        res = {"config": w.name, "nnz": w.A.nnz(), "d": d}
        for name, fn in (("fused", fused), ("unfused", unfused)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.iters):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn()
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[f"{name}_ms"] = float(np.median(ts))
        st = g.run_unfused_device(X.data_ptr(), m, X.data_ptr(), Z.data_ptr(), d, w.spec)
        res["unfused_materialised_bytes"] = int(st.aux_bytes)
        res["speedup_fused"] = res["unfused_ms"] / res["fused_ms"]
        print(json.dumps(res), flush=True)
        del g, ctx, X, Z


if __name__ == "__main__":
    main()
