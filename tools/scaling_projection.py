"""Projected multi-GPU step time per config from measured pieces (no GPU).

* compute: the slowest shard's kernel time at G shards WITH its halo stores
  (profiles/r2v_shard_balance.jsonl, tools/shard_balance.py --halo: each
  shard run alone on one B200, cost-balanced part1d, the stores going to
  local stand-in peer buffers);
* NVLink: the largest per-GPU halo ingress (profiles/r2_halo_volume_c*.jsonl)
  and egress (the same r2v lines) at the peer bandwidth a kernel's P2P
  traffic reaches (775 GB/s per direction, B300 NV18, B300_MICROARCH.md).

The exchange rides on the kernel's own stores, so a step is
max(compute, ingress / bw, egress / bw). A projection, not a measurement.

    python tools/scaling_projection.py > profiles/r3_scaling_projection.txt
"""
import json
from pathlib import Path

P = Path(__file__).resolve().parents[1] / "profiles"
BW = 775e9


def main():
    # newest measurement of every (config, shard count, halo) wins: r2v (all
    # configs), then the second-pass re-measurements (r3w configs 2 and 3, r3v, then r4c config 5)
    by_key = {}
    for name in ("r2v_shard_balance.jsonl", "r3w_shard_balance_c2.jsonl", "r3w_shard_balance_c3.jsonl", "r3v_shard_balance_c5.jsonl", "r4c_shard_balance_c5.jsonl", "r4e_shard_balance_c5_w16.jsonl"):
        f = P / name
        if not f.exists():
            continue
        for l in f.read_text().splitlines():
            if l.strip().startswith("{"):
                r = json.loads(l)
                by_key[(r["config"], r["gpus"], bool(r.get("halo_stores")))] = r
    lines = list(by_key.values())
    halo = {}
    for f in sorted(P.glob("r2_halo_volume_c*.jsonl")):
        for l in f.read_text().splitlines():
            r = json.loads(l)
            halo[(r["config"], r["gpus"])] = r
    print("config gpus t1_ms compute_ms(+halo stores) ingress_ms egress_ms step_ms projected_x "
          "| all-rows: ingress_ms projected_x")
    for c in (2, 3, 5):
        one = [r for r in lines if r["config"] == c and r["gpus"] == 1]
        if not one:
            continue
        t1 = min(r["max_ms"] for r in one)
        for g in (2, 4, 8):
            rs = [r for r in lines if r["config"] == c and r["gpus"] == g and r["halo_stores"]]
            if not rs or (c, g) not in halo:
                continue
            r = rs[0]
            comp = r["max_ms"]
            ing = halo[(c, g)]["max_ingress_bytes"] / BW * 1e3
            egr = max(r["halo_bytes_sent_per_shard"]) / BW * 1e3
            step = max(comp, ing, egr)
            ing_all = halo[(c, g)]["max_ingress_bytes_all_rows"] / BW * 1e3
            egr_all = max(halo[(c, g)]["max_ingress_bytes_all_rows"], 0) / BW * 1e3  # all rows: egress ~ slice*(G-1)
            step_all = max(comp, ing_all, egr_all)
            print(f"{c} {g} {t1:.3f} {comp:.3f} {ing:.3f} {egr:.3f} {step:.3f} {t1 / step:.2f} "
                  f"| {ing_all:.3f} {t1 / step_all:.2f}")


if __name__ == "__main__":
    main()
