"""CPU: the C-ABI library loads, exports every symbol include/fusedmm_cuda.h
declares, its host-only entry points behave like the reference, the headers
compile as C and C++, and the product fails loudly (never falls back) when no
GPU is present. No compute calls are made here."""
import ctypes as C
import re
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2011_06391_b200 import _lib
from paper_2011_06391_b200 import fusedmm as F

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "fusedmm_cuda.h"


def declared_functions():
    src = HEADER.read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fmm_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("fmm_create", "fmm_destroy", "fmm_graph_upload", "fmm_run", "fmm_iterate",
                 "fmm_last_error", "fmm_part1d", "fmm_pattern_of"):
        assert must in names


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared_functions()
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.SIGNATURES), "ctypes binding out of sync with the header"
    nm = shutil.which("nm")
    if nm:
        out = subprocess.run([nm, "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                             text=True).stdout
        exported = set(re.findall(r" T (fmm_\w+)", out))
        assert set(names) <= exported


def test_version_and_status_strings():
    L = _lib.lib()
    assert b"sm_100a" in L.fmm_version()
    assert L.fmm_status_string(_lib.FMM_E_INVAL) == b"invalid argument"
    assert L.fmm_status_string(_lib.FMM_OK) == b"ok"


@pytest.mark.parametrize("seed", range(20))
def test_part1d_abi_matches_oracle_and_reference(seed):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(0, 80))
    deg = rng.integers(0, 16, m) * (rng.random(m) < 0.8)
    row_ptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    A = F.CsrMatrix(m, 16, row_ptr, np.zeros(int(row_ptr[-1]), np.int64))
    for t in (1, 2, 3, 7, 32):
        got = F.part1d(A, t).boundaries
        assert got == oracle.oracle_part1d(row_ptr, t)
        if oracle.ref_available():
            assert got == oracle.ref_part1d(row_ptr, t)
        # soundness (test_kernel.cpp:28-42): nnz(part) <= nnz/t + max_row
        mx = int(deg.max()) if m else 0
        for i in range(t):
            assert got[i] <= got[i + 1]
            assert row_ptr[got[i + 1]] - row_ptr[got[i]] <= row_ptr[-1] / t + mx


def test_part1d_rejects_zero_workers():
    with pytest.raises(ValueError):
        F.part1d(F.CsrMatrix(1, 1, np.array([0, 1]), np.array([0])), 0)


def test_pattern_of_through_abi():
    # ops.hpp:189-203 (+ device patterns); USER never matches
    assert F.pattern_of(F.make_spec(F.App.NODE_EMBED_SIGMOID)) == F.KnownPattern.SIGMOID_EMBED
    assert F.pattern_of(F.make_spec(F.App.GCN_FORWARD)) == F.KnownPattern.SPMM_GCN
    assert F.pattern_of(F.make_spec(F.App.FR_LAYOUT)) == F.KnownPattern.FR_LAYOUT
    assert F.pattern_of(F.fr_layout_sub_spec(1.0)) == F.KnownPattern.GENERIC
    assert F.pattern_of(F.tdist_spec()) == F.KnownPattern.TDIST
    assert F.pattern_of(F.fr_attract_spec(1.0)) == F.KnownPattern.FR_ATTRACT
    s = F.OpSpec(F.Vop.USER, F.Rop.NOOP, F.Sop.SIGMOID, F.Mop.MUL, F.Aop.AMAX)
    assert F.pattern_of(s) == F.KnownPattern.GENERIC


def test_dims_checked_before_any_device_work():
    # kernel.hpp:269-282 / test_kernel.cpp:134-144
    A = F.csr_from_coo([(0, 1, 1.0)], 2, 2)
    Y = F.DenseMatrix(2, 2)
    with pytest.raises(F.InvalidArgument):
        F.fused_mm(A, F.DenseMatrix(1, 2), Y, F.make_spec(F.App.GCN_FORWARD), 1)
    with pytest.raises(F.InvalidArgument):
        F.fused_mm(A, F.DenseMatrix(2, 3), Y, F.make_spec(F.App.GCN_FORWARD), 1)
    with pytest.raises(F.InvalidArgument):
        F.fused_mm(A, F.DenseMatrix(2, 2), F.DenseMatrix(1, 2), F.make_spec(F.App.GCN_FORWARD), 1)
    with pytest.raises(F.InvalidArgument):
        F.fused_mm(A, F.DenseMatrix(2, 2), Y, F.make_spec(F.App.GCN_FORWARD), 0)
    with pytest.raises(F.InvalidArgument):
        F.make_spec(F.App.GNN_MLP)  # test_apps.cpp:44-46


def test_user_slot_is_unsupported_not_emulated():
    A = F.csr_from_coo([(0, 1, 1.0)], 2, 2)
    spec = F.make_spec(F.App.GNN_MLP, F.AppParams(mlp_vop=lambda x, y, o: None))
    with pytest.raises(F.Unsupported):
        F.fused_mm(A, F.DenseMatrix(2, 2), F.DenseMatrix(2, 2), spec, 1)


@pytest.mark.skipif(F.device_count() > 0, reason="GPU present: the no-GPU contract is moot")
def test_no_gpu_fails_loudly():
    L = _lib.lib()
    h = C.c_void_p()
    assert L.fmm_create(1, None, C.byref(h)) != _lib.FMM_OK
    A = F.csr_from_coo([(0, 1, 1.0)], 2, 2)
    with pytest.raises(F.CudaError):
        F.fused_mm(A, F.DenseMatrix(2, 2), F.DenseMatrix(2, 2), F.make_spec(F.App.GCN_FORWARD), 1)


def test_headers_compile_as_c_and_cpp(tmp_path):
    c_src = tmp_path / "t.c"
    c_src.write_text('#include "fusedmm_cuda.h"\nint main(void){fmm_opspec s={1,1,1,0,0,1.f,1.f};'
                     'int32_t p; return (int)fmm_pattern_of(&s,&p);}\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", f"-I{ROOT/'include'}", "-c", str(c_src),
                        "-o", str(tmp_path / "t.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run(["g++", "-std=c++17", "-Wall", f"-I{ROOT/'include'}", str(ROOT / "tests/cpp/wrapper_demo.cpp"),
                        f"-L{_lib.LIB_PATH.parent}", "-lfusedmm_cuda", "-o", str(tmp_path / "demo")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.parametrize("seed", range(10))
def test_part1d_weighted(seed):
    """w = 0 is exactly part1d; w > 0 balances nnz + w per row: every block's
    cost is within one row's cost of the ideal split."""
    rng = np.random.default_rng(100 + seed)
    m = int(rng.integers(1, 400))
    deg = rng.integers(0, 40, m) * (rng.random(m) < 0.7)
    row_ptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    A = F.CsrMatrix(m, m, row_ptr, np.zeros(int(row_ptr[-1]), np.int64), None)
    L = _lib.lib()
    for t in (1, 2, 3, 8):
        b = np.zeros(t + 1, np.int64)
        assert L.fmm_part1d_weighted(m, row_ptr.ctypes.data_as(C.POINTER(C.c_int64)), t, 0.0,
                                     b.ctypes.data_as(C.POINTER(C.c_int64))) == _lib.FMM_OK
        assert b.tolist() == F.part1d(A, t).boundaries
        for w in (1.0, 6.0):
            b = np.zeros(t + 1, np.int64)
            L.fmm_part1d_weighted(m, row_ptr.ctypes.data_as(C.POINTER(C.c_int64)), t, w,
                                  b.ctypes.data_as(C.POINTER(C.c_int64)))
            cost = row_ptr + w * np.arange(m + 1)
            assert b[0] == 0 and b[-1] == m and np.all(np.diff(b) >= 0)
            for i in range(1, t):
                r = b[i]
                assert cost[r] * t >= i * cost[m] - 1e-9
                assert r == 0 or cost[r - 1] * t < i * cost[m]
    assert L.fmm_part1d_weighted(m, row_ptr.ctypes.data_as(C.POINTER(C.c_int64)), 2, -1.0,
                                 np.zeros(3, np.int64).ctypes.data_as(C.POINTER(C.c_int64))) == _lib.FMM_E_INVAL


REF_INCLUDE = Path("/root/reference/proj/include")


@pytest.mark.skipif(not (REF_INCLUDE / "fusedmm" / "kernel.hpp").exists() or shutil.which("g++") is None,
                    reason="reference headers or g++ not present")
def test_cpp_dropin_compiles_against_reference_types():
    """INTEGRATION.md's claim, pinned: include/fusedmm_cuda.hpp is used from
    reference host code with the reference's own CsrMatrix / DenseMatrix /
    OpSpec / KernelStats / KernelOptions for fused_mm, update_u,
    fused_mm_specialized and tune_lane_width (tests/cpp/reference_dropin.cpp)."""
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", f"-I{ROOT / 'include'}",
                        f"-I{REF_INCLUDE}", str(ROOT / "tests" / "cpp" / "reference_dropin.cpp")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not present")
def test_cpp_wrapper_demo_builds_and_links(tmp_path):
    """The wrapper demo compiles and links against libfusedmm_cuda (runs on
    the GPU in test_gpu_ops.py::test_cpp_wrapper_runs)."""
    exe = tmp_path / "demo"
    r = subprocess.run(["g++", "-std=c++17", f"-I{ROOT / 'include'}", str(ROOT / "tests/cpp/wrapper_demo.cpp"),
                        f"-L{_lib.LIB_PATH.parent}", "-lfusedmm_cuda", f"-Wl,-rpath,{_lib.LIB_PATH.parent}",
                        "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def test_fingerprint_is_content_keyed():
    a = np.arange(1_000_003, dtype=np.int64)
    f0 = F.fingerprint(a)
    assert F.fingerprint(a.copy()) == f0          # same contents, other address
    a[777_777] += 1
    assert F.fingerprint(a) != f0                 # same address, other contents
    assert F.fingerprint(a[:10]) != F.fingerprint(a[:11])
