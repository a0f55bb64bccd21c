"""Randomised parity stress (tool, GPU): random degree distributions (empty
rows, hubs past the chunk size, column bands forced on), random d and op
specs, 1-3 shards — every case against the CPU oracle (bit-exact where the
exact scheme applies; otherwise per row within 1e-5 + four times the CPU fp32
result's own distance from fp64) and 1 shard vs t shards bitwise.

    python tests/stress_random.py --cases 200 --seed 0
"""
from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def random_graph(rng, n):
    kind = rng.integers(0, 4)
    deg = np.zeros(n, dtype=np.int64)
    if kind == 0:      # light rows, many empty
        idx = rng.choice(n, max(1, n // 3), replace=False)
        deg[idx] = rng.integers(1, 20, idx.size)
    elif kind == 1:    # power law with hubs
        deg = np.minimum((rng.pareto(1.1, n) * 3).astype(np.int64), n - 1)
        deg[rng.random(n) < 0.3] = 0
    elif kind == 2:    # a few very heavy rows + light rest
        deg[rng.choice(n, 5, replace=False)] = rng.integers(n // 2, n, 5)
        light = rng.choice(n, n // 2, replace=False)
        deg[light] = np.maximum(deg[light], rng.integers(0, 6, light.size))
    else:              # regular
        deg[:] = rng.integers(1, 40)
    row_ptr = np.concatenate([[0], np.cumsum(deg)])
    cols = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in deg if k > 0]) if deg.sum() else \
        np.zeros(0, dtype=np.int64)
    return row_ptr, cols


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=100)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    import oracle
    from paper_2011_06391_b200 import fusedmm as F
    from tests.parity import check_exact, check_tolerance

    rng = np.random.default_rng(a.seed)
    specs = [F.make_spec(F.App.NODE_EMBED_SIGMOID), F.make_spec(F.App.GCN_FORWARD),
             F.make_spec(F.App.FR_LAYOUT, F.AppParams(alpha=0.3)), F.tdist_spec(),
             F.OpSpec(F.Vop.SEL2ND, F.Rop.NOOP, F.Sop.NOOP, F.Mop.MUL, F.Aop.AMAX),
             F.OpSpec(F.Vop.ADD, F.Rop.RSUM, F.Sop.SCAL, F.Mop.MUL, F.Aop.ASUM, alpha=0.01)]
    dims = [2, 4, 8, 16, 32, 64, 100, 128, 256, 512]
    for case in range(a.cases):
        n = int(rng.choice([257, 1000, 4096, 9000]))
        d = int(rng.choice(dims))
        spec = specs[int(rng.integers(0, len(specs)))]
        bands = bool(rng.integers(0, 2))
        for k, v in (("FMM_BAND_COLS", "64" if bands else "0"), ("FMM_BAND_MINDEG", "64"), ("FMM_BAND_MINLEN", "4"),
                     ("FMM_CHUNK", str(int(rng.choice([64, 256, 1024]))))):
            os.environ[k] = v
        row_ptr, cols = random_graph(rng, n)
        weighted = bool(rng.integers(0, 2))
        vals = rng.uniform(0.1, 2.0, cols.size).astype(np.float32) if weighted else None
        A = F.CsrMatrix(n, n, row_ptr, cols, vals)
        X = F.DenseMatrix(n, d, rng.uniform(0.05, 1.0, n * d))  # positive: sums without heavy cancellation
        Zo = oracle.oracle_fused_mm(A, X, X, spec)
        Z1 = np.zeros_like(Zo)
        g = F.DeviceGraph(F.Context([0]), A)
        g.run_host(X.array, X.array, Z1, d, spec)
        tag = f"case {case}: n={n} d={d} nnz={cols.size} spec={F.pattern_of(spec).name} bands={bands} weighted={weighted}"
        try:
            if F.pattern_of(spec) == F.KnownPattern.SPMM_GCN or spec.aop == F.Aop.AMAX:
                check_exact(Z1, Zo)
            else:
                # random rows can be ill-conditioned (cancelling messages): judge the GPU
                # against fp64 with the slack the CPU fp32 result itself needs
                Z64 = oracle.oracle_fused_mm(A, X, X, spec, f64=True)
                e_gpu = np.nan_to_num(oracle.row_errors(Z1, Z64), nan=np.inf)
                e_cpu = np.nan_to_num(oracle.row_errors(Zo, Z64), nan=np.inf)
                bad = np.nonzero(e_gpu > 1e-5 + 4.0 * e_cpu)[0]
                assert bad.size == 0, f"row {int(bad[0])}: gpu-vs-fp64 {e_gpu[bad[0]]:.3e}, cpu-vs-fp64 {e_cpu[bad[0]]:.3e}"
            t = int(rng.integers(2, 4))
            gt = F.DeviceGraph(F.Context([0] * t), A)
            Zt = np.zeros_like(Zo)
            gt.run_host(X.array, X.array, Zt, d, spec)
            check_exact(Zt, Z1)
        except AssertionError as e:
            print("FAIL", tag, str(e)[:300], flush=True)
            return 1
        if case % 20 == 0:
            print("ok", tag, flush=True)
    print(f"stress ok: {a.cases} cases")
    return 0


if __name__ == "__main__":
    sys.exit(main())
