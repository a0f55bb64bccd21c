"""Exchange volume of the iterative workloads with and without the halo
masks (host-only, no GPU): for G row shards (the cost-balanced part1d the
device uses), shard s sends row r to shard q only if one of q's edges points
at r. Prints one JSON line per G: total bytes per exchange, the largest
per-GPU ingress, and the cut against sending every row to every peer.

    python tools/halo_volume.py --config 5 --gpus 2,4,8
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--gpus", default="2,4,8")
    a = ap.parse_args()
    from paper_2011_06391_b200 import configs
    from paper_2011_06391_b200 import fusedmm as F
    w = configs.get(a.config)
    A, d = w.A, w.d
    m = A.nrows
    for G in [int(x) for x in a.gpus.split(",")]:
        b = F.shard_bounds(A, G, d).boundaries
        need = []
        for q in range(G):
            cols = A.col_idx[A.row_ptr[b[q]]:A.row_ptr[b[q + 1]]]
            nq = np.zeros(m, bool)
            nq[cols] = True
            need.append(nq)
        sent = 0
        ingress = []
        for q in range(G):
            inq = 0
            for s in range(G):
                if s != q:
                    inq += int(np.count_nonzero(need[q][b[s]:b[s + 1]]))
            ingress.append(inq)
            sent += inq
        full_rows = sum((b[s + 1] - b[s]) * (G - 1) for s in range(G))
        full_ingress = [m - (b[q + 1] - b[q]) for q in range(G)]
        rec = {"config": a.config, "gpus": G, "d": d,
               "bytes_per_exchange": sent * d * 4, "bytes_per_exchange_all_rows": full_rows * d * 4,
               "cut": 1.0 - sent / full_rows,
               "max_ingress_bytes": max(ingress) * d * 4, "max_ingress_bytes_all_rows": max(full_ingress) * d * 4,
               "max_ingress_cut": 1.0 - max(ingress) / max(full_ingress)}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
