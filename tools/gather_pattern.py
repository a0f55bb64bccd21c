"""Characterise the config 2 gather stream without the FusedMM arithmetic
(tool): writes index streams for tools/probe_gather4 (file mode: plain
512-byte row gathers, summed in registers) — the real CSR column stream, the
same columns shuffled, and uniform-random rows — to see whether the R-MAT hub
skew or the fused kernel limits delivery.

    python tools/gather_pattern.py [--config 2|3]
"""
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2, choices=(2, 3))
    cfg = ap.parse_args().config
    from paper_2011_06391_b200 import configs
    w = configs.get(cfg)
    rowb = w.d * 4
    cols = w.A.col_idx.astype(np.int32)
    n = w.A.ncols
    rng = np.random.default_rng(0)
    streams = {"csr": cols, "shuffled": rng.permutation(cols),
               "uniform": rng.integers(0, n, cols.size).astype(np.int32)}
    for k, v in streams.items():
        path = f"/tmp/g{cfg}_{k}.bin"
        v.tofile(path)
        subprocess.run([str(ROOT / "tools" / "probe_gather4"), path, str(n), str(rowb)], check=True)


if __name__ == "__main__":
    main()
