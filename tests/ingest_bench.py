"""Graph construction on the host vs the device (tool; JSON lines): the
BASELINE R-MAT recipe (stream -> drop self-loops -> symmetrise -> sort ->
unique) with the host builder (libfmm_gen) and with the insertion stream
folded on the GPU (fmm_csr_sym_unique); also the reference rmat_generate
semantics (stream -> csr_from_coo) on the GPU.

    python tests/ingest_bench.py --scale 20 --ef 16 --seed 1
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    from paper_2011_06391_b200 import configs
    from paper_2011_06391_b200 import fusedmm as F
    n = 1 << a.scale
    F.csr_sym_unique_device([0], [1], 2)  # context warm-up
    t0 = time.perf_counter()
    H = configs.rmat_sym(a.scale, a.ef, a.seed)
    t_host = time.perf_counter() - t0
    t0 = time.perf_counter()
    rows, cols = configs.rmat_stream(a.scale, a.ef, a.seed)
    t_stream = time.perf_counter() - t0
    t0 = time.perf_counter()
    D = F.csr_sym_unique_device(rows, cols, n)
    t_dev = time.perf_counter() - t0
    same = bool(np.array_equal(D.row_ptr, H.row_ptr) and np.array_equal(D.col_idx, H.col_idx))
    t0 = time.perf_counter()
    R = F.csr_from_coo_device(rows, cols, None, n, n)
    t_coo = time.perf_counter() - t0
    print(json.dumps({"scale": a.scale, "edge_factor": a.ef, "stream_edges": int(rows.size), "nnz": int(D.nnz()),
                      "host_builder_s": round(t_host, 3), "stream_s": round(t_stream, 3),
                      "device_sym_unique_s": round(t_dev, 3), "device_equals_host": same,
                      "device_csr_from_coo_s": round(t_coo, 3), "rmat_generate_nnz": int(R.nnz())}), flush=True)


if __name__ == "__main__":
    main()
