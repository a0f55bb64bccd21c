"""GPU: the unfused SDDMM -> SpMM baseline (fmm_run_unfused, the device
restatement of reference.hpp:41-155) computes the same Z as the fused kernel
(within the fast scheme's tolerance) and reports the materialised-H bytes the
reference's model predicts (4 B per edge for scalar messages, 4d B per edge
for vector messages)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2011_06391_b200 import configs
from paper_2011_06391_b200 import fusedmm as F
from tests.parity import check_tolerance

pytestmark = pytest.mark.gpu


def run_both(w, spec=None):
    spec = spec or w.spec
    dev = torch.device("cuda", 0)
    X = torch.from_numpy(w.X.array).to(dev)
    Zf = torch.zeros_like(X)
    Zu = torch.zeros_like(X)
    g = F.DeviceGraph(F.Context([0]), w.A)
    from paper_2011_06391_b200 import _lib
    g.run_device(X.data_ptr(), w.A.nrows, X.data_ptr(), Zf.data_ptr(), w.d, spec,
                 flags=_lib.FMM_DEVICE_PTRS | _lib.FMM_FAST)
    st = g.run_unfused_device(X.data_ptr(), w.A.nrows, X.data_ptr(), Zu.data_ptr(), w.d, spec)
    torch.cuda.synchronize()
    return Zf.cpu().numpy(), Zu.cpu().numpy(), st


@pytest.mark.parametrize("cfg", [1, 2, 5])
def test_unfused_matches_fused_and_oracle(cfg):
    w = configs.get(cfg, small=True)
    Zf, Zu, st = run_both(w)
    Zo = oracle.oracle_fused_mm(w.A, w.X, w.X, w.spec)
    check_tolerance(Zu, Zo, w.A, w.X, w.X, w.spec)
    check_tolerance(Zf, Zo, w.A, w.X, w.X, w.spec)
    scalar = w.spec.rop != F.Rop.NOOP
    assert st.aux_bytes >= w.A.nnz() * 4 * (1 if scalar else w.d)


@pytest.mark.parametrize("spec", [
    F.OpSpec(F.Vop.MUL, F.Rop.NOOP, F.Sop.SIGMOID, F.Mop.MUL, F.Aop.ASUM),
    F.OpSpec(F.Vop.ADD, F.Rop.NORM, F.Sop.SCAL, F.Mop.MUL, F.Aop.AMAX, alpha=0.5),
    F.OpSpec(F.Vop.SUB, F.Rop.RSUM, F.Sop.NOOP, F.Mop.SEL2ND, F.Aop.ASUM),
])
def test_unfused_generic_ops(spec):
    w = configs.get(2, small=True)
    Zf, Zu, _ = run_both(w, spec)
    Zo = oracle.oracle_fused_mm(w.A, w.X, w.X, spec)
    fin = np.isfinite(Zo)
    assert np.array_equal(fin, np.isfinite(Zu))
    scale = np.maximum(np.abs(np.where(fin, Zo, 0)).max(axis=1, keepdims=True), 1e-30)
    assert np.max(np.abs(np.where(fin, Zu - Zo, 0)) / scale) < 1e-4
    if oracle.ref_available():  # the reference's own unfused pipeline
        Zr = oracle.RefCall(w.A, w.X, w.X, spec).unfused()
        assert np.max(np.abs(np.where(fin, Zu - Zr, 0)) / scale) < 1e-4
