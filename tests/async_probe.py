"""Probe (GPU): timing of the FMM_ASYNC host pipeline with torch-pinned vs
library-pinned host buffers (tuning tool)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2011_06391_b200 import configs, _lib
from paper_2011_06391_b200 import fusedmm as F
w = configs.get(2)
A, X, d, spec = w.A, w.X, w.d, w.spec
ctx = F.Context([0]); g = F.DeviceGraph(ctx, A)
def run(Xh, Zh, flags, n=10):
    for _ in range(2): g.run_host(Xh, Xh, Zh, d, spec, flags)
    ctx.sync(); t0 = time.perf_counter()
    for _ in range(n): g.run_host(Xh, Xh, Zh, d, spec, flags)
    ctx.sync(); return (time.perf_counter() - t0) / n * 1e3
tx = torch.from_numpy(X.array).pin_memory().numpy(); tz = torch.empty(X.array.shape).pin_memory().numpy()
px = F.PinnedBuffer(X.array.shape); px.array[:] = X.array; pz = F.PinnedBuffer(X.array.shape)
ux = X.array.copy(); uz = np.zeros_like(ux)
for name, (xh, zh) in {"pageable": (ux, uz), "torch-pinned": (tx, tz), "lib-pinned": (px.array, pz.array)}.items():
    print(name, f"sync {run(xh, zh, 0):.2f} ms/call  async {run(xh, zh, _lib.FMM_ASYNC):.2f} ms/call", flush=True)
