"""CPU oracle for the FusedMM hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker or the CPU baseline;
the product (paper_2011_06391_b200, libfusedmm_cuda.so) never links or calls
it and has no CPU fallback.

Two checkers:
  * libfmm_oracle.so — the C restatement (fmm_oracle.c), bit-for-bit the
    reference's fused_mm<float>/<double> (kernel.hpp:297-353);
  * libfusedmm_ref.so — the unmodified reference headers compiled in place
    (oracle/_ref, built by oracle/Makefile when /root/reference exists),
    used to pin the restatement and as the reference CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libfmm_oracle.so"
REF_SO = HERE / "_ref" / "libfusedmm_ref.so"

P64 = C.POINTER(C.c_int64)
PF = C.POINTER(C.c_float)
PD = C.POINTER(C.c_double)


class or_spec(C.Structure):
    _fields_ = [("vop", C.c_int32), ("rop", C.c_int32), ("sop", C.c_int32), ("mop", C.c_int32),
                ("aop", C.c_int32), ("alpha", C.c_double), ("k", C.c_double),
                ("mlp_wx", C.c_double), ("mlp_wy", C.c_double), ("mlp_b", C.c_double)]


def _spec(spec) -> or_spec:
    f = lambda v: float(np.float32(v))  # noqa: E731 — the reference's T=float parameters
    return or_spec(int(spec.vop), int(spec.rop), int(spec.sop), int(spec.mop), int(spec.aop),
                   f(spec.alpha), f(spec.k), f(getattr(spec, "mlp_wx", 0.0)), f(getattr(spec, "mlp_wy", 0.0)),
                   f(getattr(spec, "mlp_b", 0.0)))


_or = None
_ref = None


def oracle_lib() -> C.CDLL:
    global _or
    if _or is None:
        if not ORACLE_SO.exists():
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(str(ORACLE_SO))
        args = [C.c_int64, C.c_int64, P64, P64, None, C.c_int64, None, C.c_int64, None,
                C.POINTER(or_spec), C.c_int, C.c_int, P64, C.c_int64, None]
        L.fmm_oracle_fused_mm_f32.argtypes = [PF if a is None else a for a in args]
        L.fmm_oracle_fused_mm_f64.argtypes = [PD if a is None else a for a in args]
        L.fmm_oracle_part1d.argtypes = [C.c_int64, P64, C.c_int, P64]
        L.fmm_oracle_pattern_of.argtypes = [C.POINTER(or_spec)]
        _or = L
    return _or


def ref_available() -> bool:
    return REF_SO.exists()


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise ImportError(f"{REF_SO} missing: build with `make -C oracle` where /root/reference exists")
        L = C.CDLL(str(REF_SO))
        L.fmm_ref_prepare_f32.restype = C.c_void_p
        L.fmm_ref_prepare_f32.argtypes = [C.c_int64, C.c_int64, P64, P64, PF, C.c_int64, PF, C.c_int64,
                                          PF, C.POINTER(or_spec), C.c_int]
        L.fmm_ref_run_f32.argtypes = [C.c_void_p, C.c_int, PF, PD]
        L.fmm_ref_release_f32.argtypes = [C.c_void_p]
        L.fmm_ref_prepare_f64.restype = C.c_void_p
        L.fmm_ref_prepare_f64.argtypes = [C.c_int64, C.c_int64, P64, P64, PD, C.c_int64, PD, C.c_int64,
                                          PD, C.POINTER(or_spec), C.c_int]
        L.fmm_ref_run_f64.argtypes = [C.c_void_p, C.c_int, PD, PD]
        L.fmm_ref_release_f64.argtypes = [C.c_void_p]
        L.fmm_ref_unfused_f32.argtypes = [C.c_void_p, PF]
        L.fmm_ref_part1d.argtypes = [C.c_int64, P64, C.c_int, P64]
        L.fmm_ref_rmat.restype = C.c_int64
        L.fmm_ref_rmat.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                   P64, P64, PF]
        L.fmm_ref_pattern_of.argtypes = [C.POINTER(or_spec)]
        L.fmm_ref_read_mm.restype = C.c_int64
        L.fmm_ref_read_mm.argtypes = [C.c_char_p, P64, P64, P64, P64, PF, C.c_int64, C.c_char_p, C.c_int64]
        L.fmm_ref_write_mm.argtypes = [C.c_char_p, C.c_int64, C.c_int64, P64, P64, PF]
        L.fmm_ref_free.argtypes = [C.c_void_p]
        L.fmm_ref_rmat_sym.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                       C.POINTER(P64), C.POINTER(P64), P64]
        L.fmm_ref_normal_fill.argtypes = [PF, C.c_int64, C.c_double, C.c_uint64]
        L.fmm_ref_uniform_fill.argtypes = [PF, C.c_int64, C.c_double, C.c_double, C.c_uint64]
        L.fmm_ref_csr_from_coo.restype = C.c_int64
        L.fmm_ref_csr_from_coo.argtypes = [C.c_int64, C.c_int64, C.c_int64, P64, P64, PF, P64, P64, PF]
        _ref = L
    return _ref


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _arrs(A, X, Y, f64: bool):
    dt = np.float64 if f64 else np.float32
    Xa = np.ascontiguousarray(X.data if hasattr(X, "data") else X, dtype=dt).reshape(-1)
    Ya = Xa if (Y is X) else np.ascontiguousarray(Y.data if hasattr(Y, "data") else Y, dtype=dt).reshape(-1)
    # the values as they are now (a caller may assign A.values after building
    # an unweighted matrix); all ones is passed as NULL, which is the same a_uv
    V = np.ascontiguousarray(A.values, dtype=dt)
    if V.size == 0 or np.all(V == 1):
        V = None
    return Xa, Ya, V


def oracle_fused_mm(A, X, Y, spec, threads: int | None = None, lane_width: int = 8, rows=None,
                    f64: bool = False) -> np.ndarray:
    """fused_mm<float> (or <double> with f64=True) over all rows, or only the
    selected `rows` (output row i = rows[i]). Returns (nsel, d)."""
    L = oracle_lib()
    d = X.dim
    ny = Y.nrows
    Xa, Ya, V = _arrs(A, X, Y, f64)
    dt = np.float64 if f64 else np.float32
    sel = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    nsel = A.nrows if sel is None else sel.size
    Z = np.zeros(nsel * d, dtype=dt)
    ptr = (lambda a: a.ctypes.data_as(PD)) if f64 else (lambda a: a.ctypes.data_as(PF))
    fn = L.fmm_oracle_fused_mm_f64 if f64 else L.fmm_oracle_fused_mm_f32
    rc = fn(A.nrows, A.ncols, A.row_ptr.ctypes.data_as(P64), A.col_idx.ctypes.data_as(P64),
            None if V is None else ptr(V), d, ptr(Xa), ny, ptr(Ya), C.byref(_spec(spec)), lane_width,
            threads or host_threads(), None if sel is None else sel.ctypes.data_as(P64),
            0 if sel is None else sel.size, ptr(Z))
    if rc != 0:
        raise ValueError(f"oracle rejected the call (rc={rc})")
    return Z.reshape(nsel, d)


def oracle_part1d(row_ptr: np.ndarray, t: int) -> list:
    b = np.zeros(t + 1, np.int64)
    m = row_ptr.size - 1
    if oracle_lib().fmm_oracle_part1d(m, np.ascontiguousarray(row_ptr, np.int64).ctypes.data_as(P64), t,
                                      b.ctypes.data_as(P64)) != 0:
        raise ValueError("part1d: worker count must be >= 1")
    return [int(x) for x in b]


class RefCall:
    """The reference fusedmm::fused_mm prepared once (CsrMatrix/DenseMatrix
    built), then run/timed repeatedly: the timed region is the fused_mm call
    only, including its Z allocation and thread spawn, as in bench.hpp:98-111."""

    def __init__(self, A, X, Y, spec, lane_width: int = 8, f64: bool = False):
        L = ref_lib()
        self.f64 = f64
        Xa, Ya, V = _arrs(A, X, Y, f64)
        self._keep = (Xa, Ya, V, A)
        ptr = (lambda a: a.ctypes.data_as(PD)) if f64 else (lambda a: a.ctypes.data_as(PF))
        prep = L.fmm_ref_prepare_f64 if f64 else L.fmm_ref_prepare_f32
        self.m, self.d = A.nrows, X.dim
        self.h = prep(A.nrows, A.ncols, A.row_ptr.ctypes.data_as(P64), A.col_idx.ctypes.data_as(P64),
                      None if V is None else ptr(V), X.dim, ptr(Xa), Y.nrows, ptr(Ya),
                      C.byref(_spec(spec)), lane_width)
        if not self.h:
            raise ValueError("reference shim rejected the spec")

    def run(self, t: int | None = None, want_z: bool = True):
        L = ref_lib()
        dt = np.float64 if self.f64 else np.float32
        Z = np.zeros(self.m * self.d, dt) if want_z else None
        secs = C.c_double()
        fn = L.fmm_ref_run_f64 if self.f64 else L.fmm_ref_run_f32
        zp = None if Z is None else (Z.ctypes.data_as(PD) if self.f64 else Z.ctypes.data_as(PF))
        rc = fn(self.h, t or host_threads(), zp, C.byref(secs))
        if rc != 0:
            raise ValueError(f"reference fused_mm threw (rc={rc})")
        return (None if Z is None else Z.reshape(self.m, self.d)), secs.value

    def unfused(self) -> np.ndarray:
        Z = np.zeros(self.m * self.d, np.float32)
        if ref_lib().fmm_ref_unfused_f32(self.h, Z.ctypes.data_as(PF)) != 0:
            raise ValueError("reference unfused pipeline threw")
        return Z.reshape(self.m, self.d)

    def close(self):
        if self.h:
            (ref_lib().fmm_ref_release_f64 if self.f64 else ref_lib().fmm_ref_release_f32)(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_fused_mm(A, X, Y, spec, t: int = 1, lane_width: int = 8, f64: bool = False) -> np.ndarray:
    rc = RefCall(A, X, Y, spec, lane_width, f64)
    Z, _ = rc.run(t)
    rc.close()
    return Z


def ref_part1d(row_ptr: np.ndarray, t: int) -> list:
    b = np.zeros(t + 1, np.int64)
    m = row_ptr.size - 1
    if ref_lib().fmm_ref_part1d(m, np.ascontiguousarray(row_ptr, np.int64).ctypes.data_as(P64), t,
                                b.ctypes.data_as(P64)) != 0:
        raise ValueError("part1d: worker count must be >= 1")
    return [int(x) for x in b]


def ref_rmat(scale: int, edge_factor: int, seed: int, abc=(0.57, 0.19, 0.19)):
    """rmat_generate (rmat.hpp:24-61) as (row_ptr, col, val)."""
    L = ref_lib()
    nnz = L.fmm_ref_rmat(scale, edge_factor, *abc, seed, None, None, None)
    n = 1 << scale
    rp = np.zeros(n + 1, np.int64)
    cl = np.zeros(nnz, np.int64)
    vl = np.zeros(nnz, np.float32)
    L.fmm_ref_rmat(scale, edge_factor, *abc, seed, rp.ctypes.data_as(P64), cl.ctypes.data_as(P64),
                   vl.ctypes.data_as(PF))
    return rp, cl, vl


def ref_csr_from_coo(rows, cols, vals, m: int, n: int):
    """The unmodified reference csr_from_coo (matrix.hpp:87-140) as
    (row_ptr, col, val); raises ValueError where the reference throws."""
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    cnt = rows.size
    v = None if vals is None else np.ascontiguousarray(vals, np.float32)
    rp = np.zeros(m + 1, np.int64)
    cl = np.zeros(max(cnt, 1), np.int64)
    vl = np.zeros(max(cnt, 1), np.float32)
    nnz = ref_lib().fmm_ref_csr_from_coo(m, n, cnt, rows.ctypes.data_as(P64), cols.ctypes.data_as(P64),
                                         None if v is None else v.ctypes.data_as(PF), rp.ctypes.data_as(P64),
                                         cl.ctypes.data_as(P64), vl.ctypes.data_as(PF))
    if nnz < 0:
        raise ValueError("csr_from_coo: entry out of bounds")
    return rp, cl[:nnz], vl[:nnz]


def ref_read_matrix_market(path: str):
    """The unmodified reference read_matrix_market (mmio.hpp:23-84) as
    (m, n, row_ptr, col, val); raises ValueError(message) where it throws."""
    L = ref_lib()
    m, n = C.c_int64(), C.c_int64()
    err = C.create_string_buffer(1024)
    nnz = L.fmm_ref_read_mm(str(path).encode(), C.byref(m), C.byref(n), None, None, None, 0, err, 1024)
    if nnz < 0:
        raise ValueError(err.value.decode())
    rp = np.zeros(m.value + 1, np.int64)
    cl = np.zeros(max(nnz, 1), np.int64)
    vl = np.zeros(max(nnz, 1), np.float32)
    L.fmm_ref_read_mm(str(path).encode(), C.byref(m), C.byref(n), rp.ctypes.data_as(P64), cl.ctypes.data_as(P64),
                      vl.ctypes.data_as(PF), nnz, err, 1024)
    return m.value, n.value, rp, cl[:nnz], vl[:nnz]


def ref_write_matrix_market(path: str, m: int, n: int, row_ptr, col, val) -> None:
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cl = np.ascontiguousarray(col, np.int64)
    vl = np.ascontiguousarray(val, np.float32)
    if ref_lib().fmm_ref_write_mm(str(path).encode(), m, n, rp.ctypes.data_as(P64), cl.ctypes.data_as(P64),
                                  vl.ctypes.data_as(PF)) != 0:
        raise ValueError(f"cannot write {path}")


def oracle_csr_from_coo(rows, cols, vals, m: int, n: int):
    """CPU restatement of csr_from_coo (matrix.hpp:87-140), test
    infrastructure: bounds check (matrix.hpp:89-95); counting placement of the
    entries by row in insertion order (matrix.hpp:97-111); per row, the first
    occurrence of a column keeps its slot and later duplicates are added to it
    in insertion order with float32 arithmetic (matrix.hpp:120-131)."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    vals = np.ones(rows.size, np.float32) if vals is None else np.asarray(vals, np.float32)
    if rows.size and (rows.min() < 0 or rows.max() >= m or cols.min() < 0 or cols.max() >= n):
        raise ValueError("csr_from_coo: entry out of bounds")
    order = np.argsort(rows, kind="stable")  # counting placement == stable by row
    row_ptr = np.zeros(m + 1, np.int64)
    out_c: list = []
    out_v: list = []
    start = 0
    sr = rows[order]
    bounds = np.searchsorted(sr, np.arange(m + 1), side="left")
    for r in range(m):
        seen: dict = {}
        for p in order[bounds[r]:bounds[r + 1]]:
            c = int(cols[p])
            if c in seen:
                out_v[seen[c]] = np.float32(out_v[seen[c]] + vals[p])
            else:
                seen[c] = len(out_c)
                out_c.append(c)
                out_v.append(np.float32(vals[p]))
        row_ptr[r + 1] = len(out_c)
        start = len(out_c)
    return row_ptr, np.array(out_c, np.int64), np.array(out_v, np.float32)


def row_errors(Z_gpu: np.ndarray, Z_cpu: np.ndarray) -> np.ndarray:
    """Per-row normwise relative error ||z_gpu - z_cpu|| / ||z_cpu||, rows
    where both are zero count as 0. Non-finite values:
    elements that agree exactly (the AMAX identity -inf of an empty row, an
    inf both sides produce) are left out of the norms; a row where the GPU
    and CPU disagree on which elements are finite, or where either holds a
    NaN the other does not, is +inf (so it always fails a tolerance check)."""
    a = np.asarray(Z_gpu, np.float64)
    b = np.asarray(Z_cpu, np.float64)
    same = (a == b) | (np.isnan(a) & np.isnan(b))
    fa, fb = np.isfinite(a), np.isfinite(b)
    bad = np.any(~same & (~fa | ~fb), axis=1)
    a0 = np.where(fa & fb, a, 0.0)
    b0 = np.where(fa & fb, b, 0.0)
    num = np.linalg.norm(a0 - b0, axis=1)
    den = np.linalg.norm(b0, axis=1)
    out = np.zeros_like(num)
    nz = den > 0
    out[nz] = num[nz] / den[nz]
    out[(~nz) & (num > 0)] = np.inf
    out[bad] = np.inf
    return out


def ref_rmat_sym(scale: int, edge_factor: int, seed: int, abc=(0.57, 0.19, 0.19)):
    """BASELINE.json R-MAT recipe from the reference's own rmat_generate
    (rmat.hpp:24-61) + drop self-loops / symmetrise / sort / unique, as
    (row_ptr, col). Test infrastructure and the reference arm's inputs."""
    L = ref_lib()
    rp, cl, nnz = P64(), P64(), C.c_int64()
    if L.fmm_ref_rmat_sym(scale, edge_factor, *abc, seed, C.byref(rp), C.byref(cl), C.byref(nnz)) != 0:
        raise ValueError("rmat_sym: the reference generator threw")
    n = 1 << scale
    try:
        row_ptr = np.ctypeslib.as_array(rp, shape=(n + 1,)).copy()
        col = np.ctypeslib.as_array(cl, shape=(max(nnz.value, 1),))[:nnz.value].copy()
    finally:
        L.fmm_ref_free(C.cast(rp, C.c_void_p))
        L.fmm_ref_free(C.cast(cl, C.c_void_p))
    return row_ptr, col


def ref_normal_fill(count: int, scale: float, seed: int) -> np.ndarray:
    out = np.empty(count, np.float32)
    ref_lib().fmm_ref_normal_fill(out.ctypes.data_as(PF), count, scale, seed)
    return out


def ref_uniform_fill(count: int, lo: float, hi: float, seed: int) -> np.ndarray:
    out = np.empty(count, np.float32)
    ref_lib().fmm_ref_uniform_fill(out.ctypes.data_as(PF), count, lo, hi, seed)
    return out


class RefWorkload:
    """A BASELINE.json workload built without any repo library (reference
    arm of bench.py): duck-types the fields cpu_reference_run reads."""

    def __init__(self, name, A, X, spec, description):
        self.name, self.A, self.X, self.spec, self.description = name, A, X, spec, description

    @property
    def d(self) -> int:
        return self.X.dim


class _Csr:
    def __init__(self, m, n, row_ptr, col_idx, values=None):
        self.nrows, self.ncols = m, n
        self.row_ptr, self.col_idx = row_ptr, col_idx
        self.values = np.ones(col_idx.size, np.float32) if values is None else values
        self.unit_values = values is None

    def nnz(self) -> int:
        return int(self.row_ptr[-1])


class _Dense:
    def __init__(self, arr):
        self.nrows, self.dim = arr.shape
        self.data = arr.reshape(-1)

    @property
    def array(self):
        return self.data.reshape(self.nrows, self.dim)


class _Spec:
    def __init__(self, vop, rop, sop, mop, aop, alpha=1.0, k=1.0):
        self.vop, self.rop, self.sop, self.mop, self.aop, self.alpha, self.k = vop, rop, sop, mop, aop, alpha, k


# BASELINE.json configs 2, 3 and 5 from the reference generator
_REF_CONFIGS = {
    2: dict(scale=20, ef=16, d=128, seed=1, x="normal", name="config2_sigmoid",
            spec=(1, 1, 1, 0, 0), desc="R-MAT scale 20 ef 16 d=128 sigmoid embedding, seed 1"),
    3: dict(scale=21, ef=8, d=32, seed=2, x="uniform", name="config3_tdist",
            spec=(3, 16, 16, 16, 0), desc="R-MAT scale 21 ef 8 d=32 t-distribution, 20 iterations, seed 2"),
    5: dict(scale=24, ef=32, d=256, seed=4, x="normal", name="config5_sigmoid_large",
            spec=(1, 1, 1, 0, 0), desc="R-MAT scale 24 ef 32 d=256 sigmoid, 5 epochs, seed 4"),
}


def ref_workload(config: int, scale: int | None = None) -> RefWorkload:
    """Configs 2 / 3 / 5 built by the reference's generator (oracle/_ref)
    only. `scale` shrinks the R-MAT scale (tests)."""
    c = _REF_CONFIGS[config]
    sc = c["scale"] if scale is None else scale
    rp, cl = ref_rmat_sym(sc, c["ef"], c["seed"])
    n = 1 << sc
    if c["x"] == "normal":
        X = ref_normal_fill(n * c["d"], 0.1, c["seed"])
    else:
        X = ref_uniform_fill(n * c["d"], -10.0, 10.0, c["seed"])
    A = _Csr(n, n, rp, cl)
    return RefWorkload(c["name"], A, _Dense(X.reshape(n, c["d"])), _Spec(*c["spec"]), c["desc"])
