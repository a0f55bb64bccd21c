"""Generate golden vectors from the REFERENCE itself (oracle/_ref, the
unmodified /root/reference headers compiled by oracle/Makefile).

    make -C oracle && python tests/golden/make_golden.py

Each .npz holds a small seeded instance (CSR, X, Y, five-slot spec, lane
width) and Z = fusedmm::fused_mm<float>(A, X, Y, spec, t) as computed by the
reference. tests/test_oracle.py pins the C oracle against them on any box;
tests/test_gpu_golden.py checks the device path against them.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2011_06391_b200 import configs  # noqa: E402
from paper_2011_06391_b200 import fusedmm as F  # noqa: E402

OUT = Path(__file__).resolve().parent


def save(name, A, X, Y, spec, lane_width=8, t=3):
    Z = oracle.ref_fused_mm(A, X, Y, spec, t=t, lane_width=lane_width)
    np.savez_compressed(
        OUT / f"{name}.npz", m=A.nrows, n=A.ncols, row_ptr=A.row_ptr, col_idx=A.col_idx,
        values=A.values, unit=bool(getattr(A, "unit_values", False)), X=X.array,
        Y=Y.array, y_is_x=Y is X,
        spec=np.array([int(spec.vop), int(spec.rop), int(spec.sop), int(spec.mop), int(spec.aop)]),
        alpha=np.float32(spec.alpha), k=np.float32(spec.k),
        mlp=np.array([spec.mlp_wx, spec.mlp_wy, spec.mlp_b], np.float32), lane_width=lane_width, Z=Z)
    print(name, A.nrows, A.nnz(), X.dim, float(np.abs(Z[np.isfinite(Z)]).max(initial=0)))


def random_case(rng, m, n, d, density):
    ent = [(r, c, float(rng.uniform(0.1, 2.0))) for r in range(m) for c in range(n)
           if rng.random() < density]
    A = F.csr_from_coo(ent, m, n)
    X = F.DenseMatrix(m, d, rng.uniform(-1, 1, m * d))
    Y = F.DenseMatrix(n, d, rng.uniform(-1, 1, n * d))
    return A, X, Y


def main():
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref not built (needs /root/reference): make -C oracle")
    rng = np.random.default_rng(20110639)
    specs = {
        "sigmoid": F.make_spec(F.App.NODE_EMBED_SIGMOID),
        "gcn": F.make_spec(F.App.GCN_FORWARD),
        "fr": F.make_spec(F.App.FR_LAYOUT, F.AppParams(alpha=0.5)),
        "frsub": F.fr_layout_sub_spec(0.25),
        "tdist": F.tdist_spec(),
        "frattr": F.fr_attract_spec(1.0),
        "amax_rmul": F.OpSpec(F.Vop.ADD, F.Rop.RMUL, F.Sop.SCAL, F.Mop.SEL2ND, F.Aop.AMAX, alpha=0.7),
        "vecmsg_sigmoid_amax": F.OpSpec(F.Vop.MUL, F.Rop.NOOP, F.Sop.SIGMOID, F.Mop.MUL, F.Aop.AMAX),
        "gnn_mlp": F.make_spec(F.App.GNN_MLP, F.AppParams(mlp_vop=F.make_toy_mlp_vop(0.3, 0.7, 0.1))),
    }
    for name, spec in specs.items():
        for d in (2, 16, 64):
            A, X, Y = random_case(rng, 40, 33, d, 0.25)
            save(f"rand_{name}_d{d}", A, X, Y, spec, lane_width=int(rng.choice([4, 8, 16])))
    # d past the blocked limit (kernel.hpp:192-225) and a ragged d
    A, X, Y = random_case(rng, 12, 12, 300, 0.3)
    save("rand_sigmoid_d300", A, X, Y, specs["sigmoid"])
    A, X, Y = random_case(rng, 20, 20, 37, 0.3)
    save("rand_fr_d37", A, X, Y, specs["fr"])
    # empty rows / empty graph
    A = F.CsrMatrix(5, 5)
    X = F.DenseMatrix(5, 4, rng.uniform(-1, 1, 20))
    save("empty_graph_amax", A, X, X, specs["amax_rmul"])
    # the five BASELINE configs at desk scale (same recipes, Y = X)
    small = {1: configs.config1(n=256), 2: configs.config2(scale=8), 3: configs.config3(scale=8),
             4: configs.config4(side=16), 5: configs.config5(scale=7)}
    for c, w in small.items():
        save(f"config{c}_desk", w.A, w.X, w.X, w.spec)
    large_d(specs)


def large_d(specs=None):
    """d past the device's register-resident shapes (1024): the streamed
    kernel's cases (own seed, so the files above are unchanged)."""
    rng = np.random.default_rng(1100)
    specs = specs or {"sigmoid": F.make_spec(F.App.NODE_EMBED_SIGMOID), "gcn": F.make_spec(F.App.GCN_FORWARD),
                      "fr": F.make_spec(F.App.FR_LAYOUT, F.AppParams(alpha=0.5)), "tdist": F.tdist_spec(),
                      "vecmsg_sigmoid_amax": F.OpSpec(F.Vop.MUL, F.Rop.NOOP, F.Sop.SIGMOID, F.Mop.MUL,
                                                      F.Aop.AMAX)}
    for name in ("sigmoid", "gcn", "fr", "tdist", "vecmsg_sigmoid_amax"):
        A, X, Y = random_case(rng, 14, 12, 1100, 0.3)
        X = F.DenseMatrix(14, 1100, X.array * 0.05)
        Y = F.DenseMatrix(12, 1100, Y.array * 0.05)
        save(f"rand_{name}_d1100", A, X, Y, specs[name])


if __name__ == "__main__":
    if sys.argv[1:] == ["--large-d"]:
        large_d()
    else:
        main()
