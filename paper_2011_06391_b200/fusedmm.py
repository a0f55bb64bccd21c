"""Python mirror of the reference FusedMM interface, running on the B200 path.

Names, argument meaning and error behaviour follow the reference headers:

    index_t, DenseMatrix, CsrMatrix, csr_from_coo, validate, stats
                                        proj/include/fusedmm/matrix.hpp:15-180
    Vop/Rop/Sop/Mop/Aop, KnownPattern, OpSpec, pattern_of
                                        proj/include/fusedmm/ops.hpp:14-51,189-203
    part1d, PartitionPlan, KernelStats, KernelOptions, fused_mm,
    fused_mm_specialized                proj/include/fusedmm/kernel.hpp:16-378
    App, AppParams, make_spec, fr_layout_sub_spec, embedding_step,
    fr_layout_step, gcn_forward         proj/include/fusedmm/apps.hpp:12-88

std::invalid_argument -> InvalidArgument (a ValueError), std::logic_error ->
LogicError. `t`, the reference's worker count, is the number of GPU shards.
Every fused call goes through libfusedmm_cuda's C ABI; there is no CPU path.
"""
from __future__ import annotations

import atexit
import ctypes as C
import enum
import threading
import weakref
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import fmm_graph_info, fmm_opspec, fmm_stats

index_t = np.int64


# ----------------------------------------------------------------- errors
class FusedMMError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class LogicError(FusedMMError):
    """std::logic_error in the reference."""


class Unsupported(NotImplementedError):
    """A USER slot or shape with no device kernel (no CPU fallback)."""


class CudaError(FusedMMError):
    pass


class DeviceOutOfMemory(MemoryError):
    pass


def _raise(status: int, ctx=None, what: str = "") -> None:
    if status == _lib.FMM_OK:
        return
    msg = what
    if ctx is not None:
        e = _lib.lib().fmm_last_error(ctx)
        if e:
            msg = e.decode()
    cls = {
        _lib.FMM_E_INVAL: InvalidArgument,
        _lib.FMM_E_UNSUPPORTED: Unsupported,
        _lib.FMM_E_CUDA: CudaError,
        _lib.FMM_E_NCCL: CudaError,
        _lib.FMM_E_OOM: DeviceOutOfMemory,
        _lib.FMM_E_LOGIC: LogicError,
    }.get(status, FusedMMError)
    raise cls(msg or _lib.lib().fmm_status_string(status).decode())


# ---------------------------------------------------------------- op enums
class Vop(enum.IntEnum):
    ADD = 0
    MUL = 1
    SEL2ND = 2
    SUB = 3
    USER = 4
    MLP = 16  # device op: sigmoid(mlp_wx*x + mlp_wy*y + mlp_b) (apps.hpp:58-64)


class Rop(enum.IntEnum):
    NOOP = 0
    RSUM = 1
    RMUL = 2
    NORM = 3
    USER = 4
    SQNORM = 16  # device extension: sum of squares, no sqrt


class Sop(enum.IntEnum):
    NOOP = 0
    SIGMOID = 1
    SCAL = 2
    USER = 3
    TDIST = 16  # device extension: 1/(1+s)
    SQK = 17    # device extension: s/k


class Mop(enum.IntEnum):
    MUL = 0
    SEL2ND = 1
    USER = 2
    MUL_VOP = 16  # device extension: w = a_uv*(h*t), t the VOP output


class Aop(enum.IntEnum):
    ASUM = 0
    AMAX = 1
    USER = 2


class KnownPattern(enum.IntEnum):
    SIGMOID_EMBED = 0
    SPMM_GCN = 1
    FR_LAYOUT = 2
    GENERIC = 3
    TDIST = 16
    FR_ATTRACT = 17


@dataclass
class OpSpec:
    """OpSpec<T> (ops.hpp:22-51). USER hooks are accepted for interface parity
    but have no device kernel: fused_mm raises Unsupported for them."""
    vop: Vop = Vop.MUL
    rop: Rop = Rop.RSUM
    sop: Sop = Sop.NOOP
    mop: Mop = Mop.MUL
    aop: Aop = Aop.ASUM
    alpha: float = 1.0
    k: float = 1.0
    mlp_wx: float = 0.0
    mlp_wy: float = 0.0
    mlp_b: float = 0.0
    user_vop: Optional[Callable] = None
    user_rop: Optional[Callable] = None
    user_sop: Optional[Callable] = None
    user_mop: Optional[Callable] = None
    user_aop: Optional[Callable] = None

    def scalar_message(self) -> bool:  # ops.hpp:45
        return self.rop != Rop.NOOP

    def has_user_slot(self) -> bool:  # ops.hpp:47-50
        return (self.vop == Vop.USER or self.rop == Rop.USER or self.sop == Sop.USER
                or self.mop == Mop.USER or self.aop == Aop.USER)

    def to_c(self) -> fmm_opspec:
        return fmm_opspec(int(self.vop), int(self.rop), int(self.sop), int(self.mop),
                          int(self.aop), float(self.alpha), float(self.k), float(self.mlp_wx),
                          float(self.mlp_wy), float(self.mlp_b))


def pattern_of(spec: OpSpec) -> KnownPattern:
    """ops.hpp:189-203 (+ the two device-only patterns), via the C ABI."""
    out = C.c_int32()
    _raise(_lib.lib().fmm_pattern_of(C.byref(spec.to_c()), C.byref(out)))
    return KnownPattern(out.value)


# -------------------------------------------------------------- containers
class DenseMatrix:
    """Row-major nrows x dim float32 matrix (matrix.hpp:18-44)."""

    def __init__(self, rows: int, d: int, values=None, fill: float = 0.0):
        self.nrows = int(rows)
        self.dim = int(d)
        if values is None:
            self.data = np.full(self.nrows * self.dim, fill, dtype=np.float32)
        else:
            arr = np.ascontiguousarray(np.asarray(values, dtype=np.float32).reshape(-1))
            if arr.size != self.nrows * self.dim:
                raise InvalidArgument("DenseMatrix: data length != nrows*dim")
            if not np.all(np.isfinite(arr)):
                raise InvalidArgument("DenseMatrix: non-finite value")
            self.data = arr

    @classmethod
    def wrap(cls, arr: np.ndarray) -> "DenseMatrix":
        """Adopt a contiguous float32 (rows, d) array without the finite check."""
        a = np.ascontiguousarray(arr, dtype=np.float32)
        M = cls.__new__(cls)
        M.nrows, M.dim = int(a.shape[0]), int(a.shape[1])
        M.data = a.reshape(-1)
        return M

    @property
    def array(self) -> np.ndarray:
        return self.data.reshape(self.nrows, self.dim)

    def row(self, u: int) -> np.ndarray:
        return self.data[u * self.dim:(u + 1) * self.dim]

    def at(self, u: int, j: int) -> float:
        return float(self.data[u * self.dim + j])


@dataclass
class GraphStats:
    nrows: int = 0
    ncols: int = 0
    nnz: int = 0
    avg_degree: float = 0.0
    max_degree: int = 0


class CsrMatrix:
    """CSR adjacency with int64 indices (matrix.hpp:48-68). Per-row storage
    order is the accumulation order of every kernel."""

    def __init__(self, nrows: int = 0, ncols: int = 0, row_ptr=None, col_idx=None, values=None):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.row_ptr = (np.zeros(self.nrows + 1, dtype=np.int64) if row_ptr is None
                        else np.ascontiguousarray(row_ptr, dtype=np.int64))
        self.col_idx = (np.zeros(0, dtype=np.int64) if col_idx is None
                        else np.ascontiguousarray(col_idx, dtype=np.int64))
        if values is None:
            self.values = np.ones(self.col_idx.size, dtype=np.float32)
            self.unit_values = True
        else:
            self.values = np.ascontiguousarray(values, dtype=np.float32)
            self.unit_values = False
        self._device = {}

    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if self.row_ptr.size else 0

    def row_nnz(self, u: int) -> int:
        return int(self.row_ptr[u + 1] - self.row_ptr[u])

    def row_cols(self, u: int) -> np.ndarray:
        return self.col_idx[self.row_ptr[u]:self.row_ptr[u + 1]]

    def row_vals(self, u: int) -> np.ndarray:
        return self.values[self.row_ptr[u]:self.row_ptr[u + 1]]

    def invalidate(self) -> None:
        """Drop cached device copies after mutating the arrays in place."""
        for g in self._device.values():
            g.free()
        self._device.clear()


def csr_from_coo(entries: Sequence[tuple], m: int, n: int) -> CsrMatrix:
    """matrix.hpp:87-140: duplicates summed, per-row storage order is the
    first-occurrence order of the deduplicated entries."""
    for (r, c, _v) in entries:
        if r < 0 or r >= m or c < 0 or c >= n:
            raise InvalidArgument(f"csr_from_coo: entry ({r},{c}) out of bounds for {m}x{n}")
    rows: list[list] = [[] for _ in range(m)]
    for (r, c, v) in entries:
        rows[r].append((c, v))
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    cols: list[int] = []
    vals: list[float] = []
    for r in range(m):
        pos: dict[int, int] = {}
        for (c, v) in rows[r]:
            if c in pos:
                vals[pos[c]] = np.float32(vals[pos[c]]) + np.float32(v)
            else:
                pos[c] = len(cols)
                cols.append(c)
                vals.append(np.float32(v))
        row_ptr[r + 1] = len(cols)
    return CsrMatrix(m, n, row_ptr, np.array(cols, dtype=np.int64),
                     np.array(vals, dtype=np.float32))


def ipc_handle(dptr: int) -> tuple:
    """(CUDA IPC handle of the allocation dptr lies in, dptr's offset in it)
    (fmm_ipc_handle); the peer maps the handle and adds the offset."""
    buf = C.create_string_buffer(64)
    off = C.c_uint64()
    _raise(_lib.lib().fmm_ipc_handle(C.c_void_p(dptr), buf, C.byref(off)))
    return buf.raw, off.value


def ipc_open(handle: bytes, device: int) -> int:
    """Map another process's allocation on `device` (fmm_ipc_open)."""
    p = C.c_void_p()
    _raise(_lib.lib().fmm_ipc_open(C.create_string_buffer(handle, 64), device, C.byref(p)))
    return p.value


def ipc_close(dptr: int) -> None:
    _raise(_lib.lib().fmm_ipc_close(C.c_void_p(dptr)))


def csr_from_coo_device(rows, cols, vals, m: int, n: int, device: int = 0) -> CsrMatrix:
    """csr_from_coo (matrix.hpp:87-140) built on the GPU (fmm_csr_from_coo):
    flat arrays in insertion order; vals None means all ones. Same result and
    same InvalidArgument as the reference for an out-of-bounds entry."""
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    cnt = int(rows.size)
    if cols.size != cnt:
        raise InvalidArgument("csr_from_coo: rows and cols differ in length")
    v = None if vals is None else np.ascontiguousarray(vals, np.float32)
    rp = np.zeros(m + 1, np.int64)
    cl = np.zeros(max(cnt, 1), np.int64)
    vl = np.zeros(max(cnt, 1), np.float32)
    nnz = C.c_int64()
    st = _lib.lib().fmm_csr_from_coo(device, m, n, cnt, _i64(rows), _i64(cols),
                                     None if v is None else _f32(v), _i64(rp), _i64(cl), _f32(vl), C.byref(nnz))
    if st == _lib.FMM_E_INVAL:
        raise InvalidArgument(f"csr_from_coo: entry out of bounds for {m}x{n}")
    _raise(st)
    k = nnz.value
    return CsrMatrix(m, n, rp, cl[:k].copy(), vl[:k].copy())


class MmParseError(RuntimeError):
    """mmio.hpp:14-17: '<path>:<line>: <what>'."""


def read_matrix_market(path: str, device: int = 0) -> CsrMatrix:
    """read_matrix_market (mmio.hpp:23-84): parsed on the host with the
    reference's rules, duplicates folded by csr_from_coo on the GPU."""
    m, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    rp, cl = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
    vl = C.POINTER(C.c_float)()
    err = C.create_string_buffer(1024)
    L = _lib.lib()
    st = L.fmm_read_matrix_market(str(path).encode(), device, C.byref(m), C.byref(n), C.byref(nnz), C.byref(rp),
                                  C.byref(cl), C.byref(vl), err, 1024)
    if st == _lib.FMM_E_INVAL:
        raise MmParseError(err.value.decode())
    _raise(st)
    try:
        row_ptr = np.ctypeslib.as_array(rp, shape=(m.value + 1,)).copy()
        k = nnz.value
        col = np.ctypeslib.as_array(cl, shape=(max(k, 1),))[:k].copy()
        val = np.ctypeslib.as_array(vl, shape=(max(k, 1),))[:k].copy()
    finally:
        for ptr in (rp, cl, vl):
            L.fmm_free(C.cast(ptr, C.c_void_p))
    return CsrMatrix(m.value, n.value, row_ptr, col, val)


def write_matrix_market(A: CsrMatrix, path: str) -> None:
    """write_matrix_market (mmio.hpp:87-99)."""
    rp = np.ascontiguousarray(A.row_ptr, np.int64)
    cl = np.ascontiguousarray(A.col_idx, np.int64)
    vl = np.ascontiguousarray(A.values if A.values is not None else np.ones(cl.size), np.float32)
    st = _lib.lib().fmm_write_matrix_market(str(path).encode(), A.nrows, A.ncols, _i64(rp), _i64(cl), _f32(vl))
    if st != _lib.FMM_OK:
        raise RuntimeError(f"cannot write {path}")


def csr_sym_unique_device(rows, cols, n: int, drop_self: bool = True, symmetrize: bool = True,
                          device: int = 0) -> CsrMatrix:
    """The BASELINE.json graph recipe on the GPU (fmm_csr_sym_unique): drop
    self-loops, add both directions, sort, deduplicate; unweighted."""
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    cnt = int(rows.size)
    rp = np.zeros(n + 1, np.int64)
    cl = np.zeros(max(2 * cnt, 1), np.int64)
    nnz = C.c_int64()
    st = _lib.lib().fmm_csr_sym_unique(device, n, cnt, _i64(rows), _i64(cols), int(drop_self), int(symmetrize),
                                       _i64(rp), _i64(cl), C.byref(nnz))
    if st == _lib.FMM_E_INVAL:
        raise InvalidArgument("csr_sym_unique: vertex out of range")
    _raise(st)
    return CsrMatrix(n, n, rp, cl[:nnz.value].copy(), None)


def validate(A: CsrMatrix) -> Optional[str]:
    """matrix.hpp:143-166: first CSR invariant violation, or None."""
    if A.row_ptr.size != A.nrows + 1:
        return "row_ptr length is not nrows+1"
    if A.row_ptr[0] != 0:
        return "row_ptr[0] != 0"
    dif = np.diff(A.row_ptr)
    if np.any(dif < 0):
        return f"row_ptr not monotone at index {int(np.argmax(dif < 0)) + 1}"
    if A.col_idx.size != A.row_ptr[-1]:
        return "col_idx length != row_ptr[nrows]"
    if A.values.size != A.col_idx.size:
        return "values length != col_idx length"
    if A.col_idx.size and (A.col_idx.min() < 0 or A.col_idx.max() >= A.ncols):
        return "column index out of range"
    rows = np.repeat(np.arange(A.nrows, dtype=np.int64), dif)
    key = rows * max(A.ncols, 1) + A.col_idx
    if np.unique(key).size != key.size:
        bad = rows[np.argsort(key)][np.r_[np.diff(np.sort(key)) == 0, False]][0]
        return f"duplicate column in row {int(bad)}"
    return None


def stats(A: CsrMatrix) -> GraphStats:
    """matrix.hpp:168-180."""
    nnz = A.nnz()
    deg = np.diff(A.row_ptr)
    return GraphStats(A.nrows, A.ncols, nnz, nnz / A.nrows if A.nrows else 0.0,
                      int(deg.max()) if deg.size else 0)


# --------------------------------------------------------------- partition
@dataclass
class PartitionPlan:
    boundaries: list
    workers: int = 0


def part1d(A: CsrMatrix, t: int) -> PartitionPlan:
    """kernel.hpp:24-49 through the library's host implementation."""
    if t < 1:
        raise InvalidArgument("part1d: worker count must be >= 1")
    b = np.zeros(t + 1, dtype=np.int64)
    _raise(_lib.lib().fmm_part1d(A.nrows, _i64(A.row_ptr), t, _i64(b)))
    return PartitionPlan([int(x) for x in b], t)


def row_weight_for(d: int) -> float:
    """Per-row cost in edge-equivalents for dimension d, from fits of the
    measured shard times (tools/shard_balance.py): ~3.6 at d=32 (config 3),
    ~6 at d=128 (config 2). At d=256 (config 5 with the column bands) the
    8-shard times fit 24 edge-equivalents per non-empty row, and every row
    also costs a halo store per reading peer: w = 16 brings the slowest
    shard's compute (11.8 ms) and the largest halo egress (11.4 ms at 775
    GB/s) together, where w = 8 left the last shard sending 10.7 GB (13.8
    ms) — profiles/r4d_partition_weights.txt."""
    return 2.5 + d / 32.0 if d <= 128 else 16.0


def shard_bounds(A: CsrMatrix, t: int, d: int) -> PartitionPlan:
    """Row blocks for t GPU shards: part1d balanced on nnz + w(d) per row
    (fmm_part1d_weighted) so the shards' kernel times, not just their edge
    counts, match. Results are bitwise independent of the partition."""
    if t < 1:
        raise InvalidArgument("part1d: worker count must be >= 1")
    b = np.zeros(t + 1, dtype=np.int64)
    _raise(_lib.lib().fmm_part1d_weighted(A.nrows, _i64(A.row_ptr), t, row_weight_for(d), _i64(b)))
    return PartitionPlan([int(x) for x in b], t)


@dataclass
class KernelStats:
    """kernel.hpp:51-55 (+ device evidence)."""
    aux_bytes: int = 0
    threads: int = 0
    pattern: KnownPattern = KnownPattern.GENERIC
    exact: bool = False
    launches: int = 0
    kernel_ms: float = 0.0
    total_ms: float = 0.0

    def fill(self, s: fmm_stats) -> None:
        self.aux_bytes = int(s.aux_bytes)
        self.threads = int(s.threads)
        self.pattern = KnownPattern(s.pattern)
        self.exact = bool(s.exact)
        self.launches = int(s.launches)
        self.kernel_ms = float(s.kernel_ms)
        self.total_ms = float(s.total_ms)


@dataclass
class KernelOptions:
    """kernel.hpp:286-288. lane_width (4, 8 or 16, as in the reference)
    selects the device's gather width like the C++ wrapper does: 4 -> the
    128-bit-load shapes (variant 20), 8 / 16 -> the default 256-bit shapes;
    `variant` (tuning: any dispatcher shape id) overrides it.
    exact: None = per-pattern default, True/False = force the scheme."""
    lane_width: int = 8
    exact: Optional[bool] = None
    variant: Optional[int] = None

    def device_variant(self) -> Optional[int]:
        if self.variant is not None:
            return self.variant
        return 20 if self.lane_width == 4 else None


# ------------------------------------------------------------ ctypes utils
def _i64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _f32(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _vp(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


# ----------------------------------------------------------- device objects
# Every live native handle, so interpreter exit releases them in a defined
# order (graphs, then contexts) while CUDA is still up, instead of leaving it
# to finalisers that run in arbitrary order. The C ABI is itself order-safe:
# a context outlives its graphs (fmm_destroy defers the delete).
_live_graphs: "weakref.WeakSet" = weakref.WeakSet()
_live_contexts: "weakref.WeakSet" = weakref.WeakSet()
_shutting_down = False


@atexit.register
def _release_all() -> None:
    global _shutting_down
    for g in list(_live_graphs):
        try:
            g.free()
        except Exception:
            pass
    for c in list(_live_contexts):
        try:
            c.close()
        except Exception:
            pass
    _contexts.clear()
    _shutting_down = True


class Context:
    """An fmm_ctx: one shard (CUDA stream) per entry of `devices`. Use as a
    context manager or call close(); graphs uploaded on it stay valid until
    they are freed (the native context is deleted after its last graph)."""

    def __init__(self, devices: Sequence[int]):
        L = _lib.lib()
        self.devices = list(devices)
        arr = (C.c_int * len(self.devices))(*self.devices)
        h = C.c_void_p()
        st = L.fmm_create(len(self.devices), arr, C.byref(h))
        if st != _lib.FMM_OK:
            _raise(st, None, "fmm_create failed (no CUDA device?)")
        self.h = h
        _live_contexts.add(self)

    def __enter__(self) -> "Context":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    def sync(self) -> None:
        """Wait for every FMM_ASYNC call enqueued on this context."""
        _raise(_lib.lib().fmm_sync(self.h), self.h)

    def set_row_weight(self, w: float) -> None:
        """Row weight of the shard partition for graphs uploaded afterwards."""
        _raise(_lib.lib().fmm_set_row_weight(self.h, w), self.h)

    def set_variant(self, variant: int) -> None:
        _raise(_lib.lib().fmm_set_variant(self.h, variant), self.h)

    def variant(self) -> int:
        return int(_lib.lib().fmm_get_variant(self.h))

    def set_stream(self, shard: int, stream_handle: int) -> None:
        _raise(_lib.lib().fmm_set_stream(self.h, shard, C.c_void_p(stream_handle)), self.h)

    def close(self) -> None:
        if getattr(self, "h", None):
            _lib.lib().fmm_destroy(self.h)
            self.h = None

    def __del__(self):
        if _shutting_down:
            return
        try:
            self.close()
        except Exception:
            pass


_contexts: dict = {}
_contexts_mu = threading.Lock()
_call_mu = threading.RLock()  # fused_mm / iterate: graph-cache lookup + run


class PinnedBuffer:
    """Page-locked host memory from libfusedmm_cuda (fmm_host_alloc), viewed as
    a numpy array; the host side of FMM_ASYNC pipelined calls."""

    def __init__(self, shape, dtype=np.float32):
        self.nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        _raise(_lib.lib().fmm_host_alloc(C.byref(p), self.nbytes))
        self.ptr = p
        buf = (C.c_byte * max(self.nbytes, 1)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def close(self) -> None:
        if getattr(self, "ptr", None):
            self.array = None
            _lib.lib().fmm_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_count() -> int:
    return int(_lib.lib().fmm_device_count())


def default_context(t: int) -> Context:
    """Context with t shards over the visible GPUs (round-robin)."""
    with _contexts_mu:
        if t not in _contexts:
            n = device_count()
            if n < 1:
                raise CudaError("no CUDA device visible (libfusedmm_cuda has no CPU fallback)")
            _contexts[t] = Context([i % n for i in range(t)])
        return _contexts[t]


def _upload_values(A: CsrMatrix):
    """Edge values to upload: None (a_uv = 1, no value stream) when every
    current value is exactly 1 — decided from the array at upload time, so
    values assigned after construction are honoured."""
    v = np.ascontiguousarray(A.values, dtype=np.float32)
    if v.size and not np.all(v == 1.0):
        return v
    return None


class DeviceGraph:
    """A CSR uploaded once (fmm_graph), optionally only rows [row_begin, row_end)."""

    def __init__(self, ctx: Context, A: CsrMatrix, row_begin: int = 0, row_end: Optional[int] = None):
        self.ctx = ctx
        self.nrows, self.ncols = A.nrows, A.ncols  # no reference to A: A._device caches graphs
        rb = 0 if row_begin is None else int(row_begin)
        re = A.nrows if row_end is None else int(row_end)
        h = C.c_void_p()
        v = _upload_values(A)
        st = _lib.lib().fmm_graph_upload(ctx.h, A.nrows, A.ncols, _i64(A.row_ptr), _i64(A.col_idx),
                                         None if v is None else _f32(v), rb, re, C.byref(h))
        _raise(st, ctx.h)
        self.h = h
        self.row_begin, self.row_end = rb, re
        _live_graphs.add(self)

    def __enter__(self) -> "DeviceGraph":
        return self

    def __exit__(self, *exc) -> None:
        self.free()

    def update_values(self, values: Optional[np.ndarray]) -> None:
        """New a_uv for the same structure (fmm_graph_update_values); values
        is the full nnz array of the uploaded CSR, None = all ones."""
        v = None if values is None else np.ascontiguousarray(values, np.float32)
        _raise(_lib.lib().fmm_graph_update_values(self.h, None if v is None else _f32(v)), self.ctx.h)

    def column_use(self) -> np.ndarray:
        """need[c] = 1 for every column this graph's edges point at."""
        need = np.zeros(max(self.ncols, 1), np.uint8)
        _raise(_lib.lib().fmm_graph_column_use(self.h, C.c_void_p(need.ctypes.data)), self.ctx.h)
        return need[:self.ncols]

    def set_peer_mask(self, mask: Optional[np.ndarray], npeer: int) -> None:
        """Halo mask for fmm_run_peers: bit q of mask[r] = peer slot q reads
        row row_begin + r (None clears it: every row to every peer)."""
        if mask is None:
            _raise(_lib.lib().fmm_graph_set_peer_mask(self.h, None, npeer), self.ctx.h)
            return
        m = np.ascontiguousarray(mask, np.uint8)
        if m.size != self.row_end - self.row_begin:
            raise InvalidArgument("set_peer_mask: one byte per row of the graph")
        _raise(_lib.lib().fmm_graph_set_peer_mask(self.h, C.c_void_p(m.ctypes.data), npeer), self.ctx.h)

    def info(self) -> fmm_graph_info:
        I = fmm_graph_info()
        _raise(_lib.lib().fmm_graph_get_info(self.h, C.byref(I)))
        return I

    def shard_bounds(self) -> list:
        I = self.info()
        b = np.zeros(I.shards + 1, dtype=np.int64)
        _raise(_lib.lib().fmm_graph_shard_bounds(self.h, _i64(b)))
        return [int(x) for x in b]

    def run_host(self, X: np.ndarray, Y: np.ndarray, Z: np.ndarray, d: int, spec: OpSpec,
                 flags: int = 0) -> fmm_stats:
        s = fmm_stats()
        st = _lib.lib().fmm_run(self.ctx.h, self.h, C.byref(spec.to_c()), d, _vp(X),
                                Y.shape[0] if Y.ndim == 2 else Y.size // max(d, 1), _vp(Y), _vp(Z),
                                flags, C.byref(s))
        _raise(st, self.ctx.h)
        return s

    def run_device(self, x_ptr: int, ny: int, y_ptr: int, z_ptr: int, d: int, spec: OpSpec,
                   flags: int = _lib.FMM_DEVICE_PTRS | _lib.FMM_ASYNC,
                   stats: Optional[fmm_stats] = None) -> None:
        st = _lib.lib().fmm_run(self.ctx.h, self.h, C.byref(spec.to_c()), d, C.c_void_p(x_ptr), ny,
                                C.c_void_p(y_ptr), C.c_void_p(z_ptr), flags,
                                C.byref(stats) if stats is not None else None)
        _raise(st, self.ctx.h)

    def run_device_peers(self, x_ptr: int, ny: int, y_ptr: int, z_ptr: int, d: int, spec: OpSpec,
                         peer_ptrs: Sequence[int], flags: int = _lib.FMM_DEVICE_PTRS | _lib.FMM_ASYNC,
                         stats: Optional[fmm_stats] = None) -> None:
        """run_device with every final z row also stored into the peer
        buffers (fmm_run_peers): the fused cross-process exchange."""
        arr = (C.c_void_p * max(len(peer_ptrs), 1))(*[C.c_void_p(p) for p in peer_ptrs])
        st = _lib.lib().fmm_run_peers(self.ctx.h, self.h, C.byref(spec.to_c()), d, C.c_void_p(x_ptr), ny,
                                      C.c_void_p(y_ptr), C.c_void_p(z_ptr), arr, len(peer_ptrs), flags,
                                      C.byref(stats) if stats is not None else None)
        _raise(st, self.ctx.h)

    def run_unfused_device(self, x_ptr: int, ny: int, y_ptr: int, z_ptr: int, d: int, spec: OpSpec,
                           flags: int = _lib.FMM_DEVICE_PTRS) -> fmm_stats:
        """The unfused SDDMM -> SpMM baseline (fmm_run_unfused)."""
        s = fmm_stats()
        st = _lib.lib().fmm_run_unfused(self.ctx.h, self.h, C.byref(spec.to_c()), d, C.c_void_p(x_ptr), ny,
                                        C.c_void_p(y_ptr), C.c_void_p(z_ptr), flags, C.byref(s))
        _raise(st, self.ctx.h)
        return s

    def iterate_host(self, X: np.ndarray, d: int, spec: OpSpec, iters: int, flags: int = 0) -> fmm_stats:
        s = fmm_stats()
        st = _lib.lib().fmm_iterate(self.ctx.h, self.h, C.byref(spec.to_c()), d, _vp(X), iters, flags,
                                    C.byref(s))
        _raise(st, self.ctx.h)
        return s

    def free(self) -> None:
        if getattr(self, "h", None):
            _lib.lib().fmm_graph_free(self.h)
            self.h = None

    def __del__(self):
        if _shutting_down:
            return
        try:
            self.free()
        except Exception:
            pass


def fingerprint(a: np.ndarray) -> int:
    """64-bit content fingerprint of an array (fmm_fingerprint)."""
    a = np.ascontiguousarray(a)
    return int(_lib.lib().fmm_fingerprint(C.c_void_p(a.ctypes.data), a.nbytes))


def _device_graph(A: CsrMatrix, t: int, d: int = 0) -> DeviceGraph:
    """The uploaded copy of A for t shards, keyed on A's CONTENTS: the
    reference reads A afresh on every fused_mm (kernel.hpp:297-353), so a CSR
    rebuilt at the same addresses, or edited in place, is re-uploaded (or,
    when only the values changed, gets its values replaced)."""
    skey = (t, A.nrows, A.ncols, A.nnz(), fingerprint(A.row_ptr), fingerprint(A.col_idx))
    vals = _upload_values(A)
    vkey = None if vals is None else fingerprint(vals)
    g = A._device.get(t)
    if g is not None and g._skey == skey:
        if g._vkey != vkey:
            g.update_values(vals)
            g._vkey = vkey
        return g
    if g is not None:
        g.free()
    ctx = default_context(t)
    if t > 1:  # shards balanced on nnz + the per-row cost for this d
        ctx.set_row_weight(row_weight_for(d) if d > 0 else 0.0)
    g = DeviceGraph(ctx, A)
    g._skey, g._vkey = skey, vkey
    A._device[t] = g
    return g


# ------------------------------------------------------------- entry points
def _check_dims(A: CsrMatrix, X: DenseMatrix, Y: DenseMatrix) -> None:
    """kernel.hpp:269-282, same messages."""
    if X.nrows != A.nrows:
        raise InvalidArgument("fused_mm: X.nrows != A.nrows")
    if X.dim != Y.dim:
        raise InvalidArgument("fused_mm: X.dim != Y.dim")
    if Y.nrows < A.ncols and A.nnz() > 0 and Y.nrows < int(A.col_idx.max()) + 1:
        raise InvalidArgument("fused_mm: Y has too few rows")


def _flags(opts: Optional[KernelOptions]) -> int:
    if opts is None:
        return 0
    if opts.lane_width not in (4, 8, 16):
        raise InvalidArgument("KernelOptions.lane_width must be 4, 8 or 16")
    if opts.exact is True:
        return _lib.FMM_EXACT
    if opts.exact is False:
        return _lib.FMM_FAST
    return 0


def fused_mm(A: CsrMatrix, X: DenseMatrix, Y: DenseMatrix, spec: OpSpec, t: int = 1,
             stats: Optional[KernelStats] = None, opts: Optional[KernelOptions] = None) -> DenseMatrix:
    """kernel.hpp:297-353 on the B200: Z[u,:] = update_u(a_u, x_u, Y, spec)
    for every row, one pass, no per-edge message buffer. t = GPU shards."""
    _check_dims(A, X, Y)
    if t < 1:
        raise InvalidArgument("fused_mm: t must be >= 1")
    if spec.has_user_slot():
        raise Unsupported("fused_mm: USER slot has no device kernel (no CPU fallback)")
    flags = _flags(opts)
    Z = DenseMatrix(A.nrows, X.dim)
    if A.nrows == 0:
        if stats is not None:
            stats.threads, stats.pattern = t, pattern_of(spec)
        return Z
    Xd = X.data if X.data.size else np.zeros(1, np.float32)
    Yd = Y.data if Y.data.size else np.zeros(1, np.float32)
    s = fmm_stats()
    prev = None
    want = opts.device_variant() if opts is not None else None
    # lookup + run under one lock: another thread's call on the same A must
    # not replace (free) the cached graph between the two
    with _call_mu:
        g = _device_graph(A, t, X.dim)
        if want is not None:
            prev = g.ctx.variant()
            g.ctx.set_variant(want)
        try:
            st = _lib.lib().fmm_run(g.ctx.h, g.h, C.byref(spec.to_c()), X.dim, _vp(Xd), Y.nrows,
                                    _vp(Xd) if Y is X else _vp(Yd), _vp(Z.data), flags, C.byref(s))
        finally:
            if prev is not None:
                g.ctx.set_variant(prev)
        _raise(st, g.ctx.h)
    if stats is not None:
        stats.fill(s)
    return Z


def fused_mm_specialized(pattern: KnownPattern, A: CsrMatrix, X: DenseMatrix, Y: DenseMatrix,
                         alpha: float, t: int = 1, opts: Optional[KernelOptions] = None) -> DenseMatrix:
    """kernel.hpp:356-378."""
    if pattern == KnownPattern.SIGMOID_EMBED:
        spec = OpSpec(Vop.MUL, Rop.RSUM, Sop.SIGMOID, Mop.MUL, Aop.ASUM)
    elif pattern == KnownPattern.SPMM_GCN:
        spec = OpSpec(Vop.SEL2ND, Rop.NOOP, Sop.NOOP, Mop.MUL, Aop.ASUM)
    elif pattern == KnownPattern.FR_LAYOUT:
        spec = OpSpec(Vop.ADD, Rop.NORM, Sop.SCAL, Mop.MUL, Aop.ASUM, alpha=alpha)
    elif pattern == KnownPattern.TDIST:
        spec = tdist_spec()
    elif pattern == KnownPattern.FR_ATTRACT:
        spec = fr_attract_spec(alpha if alpha else 1.0)
    else:
        raise InvalidArgument("fused_mm_specialized: pattern has no fast path")
    return fused_mm(A, X, X if Y is X else Y, spec, t, None, opts)


# shape variants the dispatcher defines (fmm_dispatch.cuh); unknown ones for a
# given d fall back to its default, so timing them is harmless
SHAPE_VARIANTS = (-1, 0, 1, 2, 3, 4, 5, 6, 7, 20, 21, 22, 23, 24)


def _time_opts(A, X, Y, spec, t, opts, repeats) -> float:
    fused_mm(A, X, Y, spec, t, None, opts)  # warm-up
    ms = 0.0
    for _ in range(repeats):
        st = KernelStats()
        fused_mm(A, X, Y, spec, t, st, opts)
        ms += st.kernel_ms
    return ms


def tune_lane_width(A: CsrMatrix, X: DenseMatrix, Y: DenseMatrix, spec: OpSpec, t: int = 1,
                    repeats: int = 3) -> int:
    """kernel.hpp:382-402 on the device, same contract as the reference:
    times the lane widths {4, 8, 16} (device time of the fused kernels after
    a warm-up; 4 = 128-bit gathers, 8 / 16 = the default 256-bit shapes) and
    returns the fastest width, to pass back as KernelOptions(lane_width=...)."""
    best, best_ms = 8, float("inf")
    for w in (4, 8, 16):
        ms = _time_opts(A, X, Y, spec, t, KernelOptions(lane_width=w), repeats)
        if ms < best_ms:
            best, best_ms = w, ms
    return best


def tune_variant(A: CsrMatrix, X: DenseMatrix, Y: DenseMatrix, spec: OpSpec, t: int = 1,
                 repeats: int = 3) -> int:
    """Device extension (tuning): the fastest dispatcher shape id among
    SHAPE_VARIANTS, for KernelOptions(variant=...)."""
    best, best_ms = -1, float("inf")
    for v in SHAPE_VARIANTS:
        ms = _time_opts(A, X, Y, spec, t, KernelOptions(variant=v), repeats)
        if ms < best_ms:
            best, best_ms = v, ms
    return best


def iterate(A: CsrMatrix, X: DenseMatrix, spec: OpSpec, iters: int, t: int = 1,
            stats: Optional[KernelStats] = None, opts: Optional[KernelOptions] = None) -> DenseMatrix:
    """iters fused calls with X <- Z (Y = X), resident on the device; with
    t > 1 shards the Z slices are exchanged between shards each iteration."""
    if A.nrows != A.ncols or X.nrows != A.nrows:
        raise InvalidArgument("iterate: needs a square A and X.nrows == A.nrows")
    if spec.has_user_slot():
        raise Unsupported("iterate: USER slot has no device kernel")
    out = DenseMatrix.wrap(X.array.copy())
    if A.nrows == 0:
        return out
    with _call_mu:
        g = _device_graph(A, t, X.dim)
        s = g.iterate_host(out.data, X.dim, spec, iters, _flags(opts))
    if stats is not None:
        stats.fill(s)
    return out


# ------------------------------------------------------------------ apps
class App(enum.IntEnum):
    FR_LAYOUT = 0
    NODE_EMBED_SIGMOID = 1
    GCN_FORWARD = 2
    GNN_MLP = 3


@dataclass
class AppParams:
    alpha: float = 1.0
    mlp_vop: Optional[Callable] = None


def make_spec(app: App, params: Optional[AppParams] = None) -> OpSpec:
    """apps.hpp:22-45."""
    params = params or AppParams()
    if app == App.FR_LAYOUT:
        return OpSpec(Vop.ADD, Rop.NORM, Sop.SCAL, Mop.MUL, Aop.ASUM, alpha=params.alpha)
    if app == App.NODE_EMBED_SIGMOID:
        return OpSpec(Vop.MUL, Rop.RSUM, Sop.SIGMOID, Mop.MUL, Aop.ASUM)
    if app == App.GCN_FORWARD:
        return OpSpec(Vop.SEL2ND, Rop.NOOP, Sop.NOOP, Mop.MUL, Aop.ASUM)
    if app == App.GNN_MLP:
        if params.mlp_vop is None:
            raise InvalidArgument("make_spec: GNN_MLP needs a user-provided MLP function")
        if isinstance(params.mlp_vop, ToyMLP):
            # the toy hook has a device op; any other callable stays a USER slot
            m = params.mlp_vop
            return OpSpec(Vop.MLP, Rop.NOOP, Sop.SIGMOID, Mop.MUL, Aop.AMAX, mlp_wx=m.w_x, mlp_wy=m.w_y,
                          mlp_b=m.bias)
        return OpSpec(Vop.USER, Rop.NOOP, Sop.SIGMOID, Mop.MUL, Aop.AMAX, user_vop=params.mlp_vop)
    raise InvalidArgument("make_spec: unknown app")


@dataclass
class ToyMLP:
    """make_toy_mlp_vop (apps.hpp:58-64): out[j] = sigmoid(w_x*x[j] + w_y*y[j]
    + bias). Callable like the reference lambda, and recognised by make_spec
    as the device op Vop.MLP."""
    w_x: float
    w_y: float
    bias: float

    def __call__(self, x, y, out):
        x = np.asarray(x, np.float32)
        y = np.asarray(y, np.float32)
        pre = (np.float32(self.w_x) * x + np.float32(self.w_y) * y) + np.float32(self.bias)
        out[:] = (np.float32(1) / (np.float32(1) + np.exp(-pre))).astype(np.float32)


def make_toy_mlp_vop(w_x: float, w_y: float, bias: float) -> ToyMLP:
    """apps.hpp:58-64."""
    return ToyMLP(w_x, w_y, bias)


def fr_layout_sub_spec(alpha: float) -> OpSpec:
    """apps.hpp:49-54."""
    return OpSpec(Vop.SUB, Rop.NORM, Sop.SCAL, Mop.MUL, Aop.ASUM, alpha=alpha)


def tdist_spec() -> OpSpec:
    """Config 3 t-distribution layout: t = x_u - x_v, s = |t|^2,
    h = 1/(1+s), w = a_uv*(h*t), summed (the reference's USER-VOP lambda)."""
    return OpSpec(Vop.SUB, Rop.SQNORM, Sop.TDIST, Mop.MUL_VOP, Aop.ASUM)


def fr_attract_spec(k: float = 1.0) -> OpSpec:
    """Config 4 FR-attractive: h = |x_u - x_v|^2 / k scales the difference."""
    return OpSpec(Vop.SUB, Rop.SQNORM, Sop.SQK, Mop.MUL_VOP, Aop.ASUM, k=k)


def embedding_step(A: CsrMatrix, X: DenseMatrix, Y: DenseMatrix, t: int = 1) -> DenseMatrix:
    """apps.hpp:67-71."""
    return fused_mm(A, X, Y, make_spec(App.NODE_EMBED_SIGMOID), t)


def fr_layout_step(A: CsrMatrix, X: DenseMatrix, Y: DenseMatrix, alpha: float, t: int = 1) -> DenseMatrix:
    """apps.hpp:74-80."""
    return fused_mm(A, X, Y, make_spec(App.FR_LAYOUT, AppParams(alpha=alpha)), t)


def gcn_forward(A: CsrMatrix, Y: DenseMatrix, t: int = 1) -> DenseMatrix:
    """apps.hpp:83-88 (X is a zero matrix; SEL2ND never reads it)."""
    X = DenseMatrix(A.nrows, Y.dim)
    return fused_mm(A, X, Y, make_spec(App.GCN_FORWARD), t)
