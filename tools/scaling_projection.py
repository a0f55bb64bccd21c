"""Projected multi-GPU step time per config from measured pieces (no GPU):
the slowest shard's kernel time at G shards (profiles/r06_shard_balance.jsonl,
each shard run alone on one B200, cost-balanced part1d) and the largest
per-GPU halo ingress (profiles/r2_halo_volume_c*.jsonl) over NVLink at the
peer bandwidth a kernel's P2P traffic reaches (775 GB/s, measured on B300
NV18, B300_MICROARCH.md). The exchange rides on the kernel's own stores, so
a step is max(compute, ingress / bandwidth). A projection, not a measurement.

    python tools/scaling_projection.py > profiles/r2_scaling_projection.txt
"""
import json
from pathlib import Path

P = Path(__file__).resolve().parents[1] / "profiles"
BW = 775e9


def main():
    bal = [json.loads(l) for l in (P / "r06_shard_balance.jsonl").read_text().splitlines() if l.strip()]
    halo = {}
    for f in sorted(P.glob("r2_halo_volume_c*.jsonl")):
        for l in f.read_text().splitlines():
            r = json.loads(l)
            halo[(r["config"], r["gpus"])] = r
    print("config gpus compute_ms compute_x ingress_ms(halo) ingress_ms(all rows) projected_x(halo) projected_x(all rows)")
    for c in (2, 3, 5):
        pick = {b["gpus"]: b for b in bal if b["config"] == c and b["partition"] == "weighted"}
        if 1 not in pick:
            continue
        t1 = pick[1]["max_ms"]
        for g in (2, 4, 8):
            if g not in pick or (c, g) not in halo:
                continue
            comp = pick[g]["max_ms"]
            h = halo[(c, g)]
            ing = h["max_ingress_bytes"] / BW * 1e3
            ing_all = h["max_ingress_bytes_all_rows"] / BW * 1e3
            print(f"{c} {g} {comp:.3f} {t1 / comp:.2f} {ing:.3f} {ing_all:.3f} "
                  f"{t1 / max(comp, ing):.2f} {t1 / max(comp, ing_all):.2f}")


if __name__ == "__main__":
    main()
