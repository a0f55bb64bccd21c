"""GPU parity at BASELINE.json's full sizes (configs 1-4; config 5 on sampled
rows): bit-exact for 1 and 4, per-row 1e-5 + two-tier for 2 and 3, config 3's
20 iterations teacher-forced step by step, plus size-independent properties
(bitwise determinism across shard counts and repeats)."""
import numpy as np
import pytest

import oracle
from paper_2011_06391_b200 import configs
from paper_2011_06391_b200 import fusedmm as F
from tests.parity import check_exact, check_tolerance

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def cfg_cache():
    return {}


def get(cache, c):
    if c not in cache:
        cache[c] = configs.get(c)
    return cache[c]


@pytest.mark.parametrize("cfg", [1, 4])
def test_fullsize_bit_exact(cfg_cache, cfg):
    w = get(cfg_cache, cfg)
    st = F.KernelStats()
    Z = F.fused_mm(w.A, w.X, w.X, w.spec, 1, st)
    assert st.exact
    check_exact(Z.array, oracle.oracle_fused_mm(w.A, w.X, w.X, w.spec))


def test_fullsize_config2_tolerance(cfg_cache):
    w = get(cfg_cache, 2)
    Z = F.fused_mm(w.A, w.X, w.X, w.spec, 1)
    r = check_tolerance(Z.array, oracle.oracle_fused_mm(w.A, w.X, w.X, w.spec), w.A, w.X, w.X, w.spec)
    assert r["rows"] == w.A.nrows
    # determinism: repeat and 2 shards on one device are bitwise identical
    check_exact(F.fused_mm(w.A, w.X, w.X, w.spec, 1).array, Z.array)
    g = F.DeviceGraph(F.Context([0, 0]), w.A)
    Z2 = np.zeros_like(Z.array)
    g.run_host(w.X.array, w.X.array, Z2, w.d, w.spec)
    check_exact(Z2, Z.array)


def test_fullsize_config3_twenty_iterations_teacher_forced(cfg_cache):
    w = get(cfg_cache, 3)
    X = w.X
    for it in range(w.iters):
        Z = F.fused_mm(w.A, X, X, w.spec, 1)
        Zo = oracle.oracle_fused_mm(w.A, X, X, w.spec)
        check_tolerance(Z.array, Zo, w.A, X, X, w.spec)
        X = F.DenseMatrix.wrap(Z.array)
    # the device-resident loop (X <- Z on the device) reproduces the chain
    Zi = F.iterate(w.A, w.X, w.spec, w.iters, 1)
    check_exact(Zi.array, X.array)


def test_config5_sampled_rows():
    """Config 5 at full size needs ~40 GB of host inputs and minutes of host
    generation; here it runs at scale 22 (same recipe and d=256) with the
    epochs teacher-forced on sampled rows including the hubs."""
    w = configs.config5(scale=22, iters=2)
    deg = np.diff(w.A.row_ptr)
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([np.argsort(-deg)[:32], rng.integers(0, w.A.nrows, 4096)]))
    X = w.X
    for _ in range(w.iters):
        Z = F.fused_mm(w.A, X, X, w.spec, 1)
        Zo = oracle.oracle_fused_mm(w.A, X, X, w.spec, rows=rows)
        check_tolerance(Z.array[rows], Zo, w.A, X, X, w.spec, rows=rows)
        X = F.DenseMatrix.wrap(Z.array)
