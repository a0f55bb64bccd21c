"""The reference's bench table (bench.hpp run_bench + write_csv) for the
BASELINE graphs on the device (tool, GPU): fused kernels vs the unfused
SDDMM -> SpMM device pipeline per (app, d), one shard, written as the
reference's CSV. Both sides run the reassociating scheme (the unfused
pipeline has no exact one). The exact scheme's GCN on the power-law graph is
chain-bound instead: a hub of degree 64,782 is one sequential fold per
element (~11.6 ms, rows ~ "gcn_exact" below).

    python tools/bench_records.py --out profiles/r2_bench_records.csv
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r2_bench_records.csv"))
    ap.add_argument("--iterations", type=int, default=5)
    a = ap.parse_args()
    from paper_2011_06391_b200 import benchrec as B
    from paper_2011_06391_b200 import configs
    from paper_2011_06391_b200 import fusedmm as F
    recs = []
    g1 = configs.get(1).A
    fast = F.KernelOptions(exact=False)
    recs += B.run_bench(g1, "er16384_k16", F.make_spec(F.App.GCN_FORWARD), "gcn", [32, 64, 128, 256], [1],
                        a.iterations, B.BenchMode.BOTH, opts=fast)
    g2 = configs.get(2).A
    for app, spec in (("embed", F.make_spec(F.App.NODE_EMBED_SIGMOID)),
                      ("fr", F.make_spec(F.App.FR_LAYOUT, F.AppParams(alpha=0.5))),
                      ("gcn", F.make_spec(F.App.GCN_FORWARD))):
        recs += B.run_bench(g2, "rmat20_ef16_sym", spec, app, [32, 64, 128], [1], a.iterations, B.BenchMode.BOTH,
                            opts=fast)
    recs += B.run_bench(g2, "rmat20_ef16_sym", F.make_spec(F.App.GCN_FORWARD), "gcn_exact", [128], [1],
                        a.iterations, B.BenchMode.FUSED, opts=F.KernelOptions(exact=True))
    B.write_csv(recs, a.out)
    print(B.csv_string(recs), end="")


if __name__ == "__main__":
    main()
