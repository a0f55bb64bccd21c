"""The five BASELINE.json workloads as seeded synthetic inputs.

Every config is synthetic (BASELINE.json names no dataset). Graphs and X are
generated on the host by libfmm_gen (C++), deterministically from the seed, so
the device path and the CPU oracle consume identical buffers. Recipes:
SURVEY.md §8(d) and DESIGN.md §"Inputs". `scale_down` shrinks the R-MAT scale
/ lattice side / row count for parity tests that must finish in seconds on
the CPU oracle while keeping each config's shape and value distribution.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .fusedmm import CsrMatrix, DenseMatrix, OpSpec, fr_attract_spec, make_spec, App, tdist_spec

RMAT_ABC = (0.57, 0.19, 0.19)  # d = 0.05


@dataclass
class Workload:
    name: str
    A: CsrMatrix
    X: DenseMatrix
    spec: OpSpec
    iters: int
    weighted: bool
    exact: bool          # parity contract: bit-exact vs the reference
    description: str

    @property
    def d(self) -> int:
        return self.X.dim

    def nonempty_rows(self) -> int:
        return int(np.count_nonzero(np.diff(self.A.row_ptr)))

    def alg_bytes(self) -> int:
        """B_alg of SURVEY.md §8(d): 8(m+1) row_ptr + 4 nnz int32 columns
        + 4 nnz a_uv (weighted only) + 4 d nnz gathers + 4 d m_nz x_u reads
        (when VOP reads x) + 4 d m Z writes."""
        m, nnz, d = self.A.nrows, self.A.nnz(), self.d
        reads_x = self.spec.vop != 2  # SEL2ND never reads x_u
        b = 8 * (m + 1) + 4 * nnz + 4 * d * nnz + 4 * d * m
        if self.weighted:
            b += 4 * nnz
        if reads_x:
            b += 4 * d * self.nonempty_rows()
        return b


def _take(ptr, count: int, dtype) -> np.ndarray:
    arr = np.ctypeslib.as_array(ptr, shape=(max(count, 1),))[:count].astype(dtype, copy=True)
    _lib.gen().fmmgen_free(ptr)
    return arr


def rmat_sym(scale: int, edge_factor: int, seed: int) -> CsrMatrix:
    G = _lib.gen()
    rp = C.POINTER(C.c_int64)()
    cl = C.POINTER(C.c_int64)()
    nnz = C.c_int64()
    rc = G.fmmgen_rmat_sym(scale, edge_factor, *RMAT_ABC, seed, C.byref(rp), C.byref(cl), C.byref(nnz))
    if rc != 0:
        raise ValueError("rmat_sym: bad parameters")
    n = 1 << scale
    return CsrMatrix(n, n, _take(rp, n + 1, np.int64), _take(cl, nnz.value, np.int64), None)


def rmat_generate(scale: int, edge_factor: int = 16, seed: int = 1, device: int = 0) -> CsrMatrix:
    """rmat_generate (rmat.hpp:24-61): the seeded insertion stream (host,
    one sequential mt19937_64) folded by csr_from_coo on the GPU — self-loops
    kept, duplicates summed into values > 1. Bitwise equal to the reference."""
    from .fusedmm import csr_from_coo_device
    rows, cols = rmat_stream(scale, edge_factor, seed)
    n = 1 << scale
    return csr_from_coo_device(rows, cols, None, n, n, device)


def rmat_device(scale: int, edge_factor: int, seed: int, recipe: int = 1, device: int = 0):
    """The R-MAT graphs built entirely on the GPU (fmm_rmat_device): the
    insertion stream from jump-ahead mt19937_64 sub-streams, then recipe 1
    (BASELINE: drop self-loops, symmetrise, sort, unique — equals rmat_sym),
    recipe 0 (csr_from_coo: equals the reference's rmat_generate), or
    recipe 2 (the raw stream as (rows, cols))."""
    from .fusedmm import InvalidArgument, _raise
    n = 1 << scale
    ne = edge_factor << scale
    L = _lib.lib()
    P64 = C.POINTER(C.c_int64)
    nnz = C.c_int64()
    if recipe == 2:
        rows = np.zeros(max(ne, 1), np.int64)
        cols = np.zeros(max(ne, 1), np.int64)
        st = L.fmm_rmat_device(device, scale, edge_factor, *RMAT_ABC, seed, 2, None, None, None,
                               rows.ctypes.data_as(P64), cols.ctypes.data_as(P64), C.byref(nnz))
        if st == _lib.FMM_E_INVAL:
            raise InvalidArgument("rmat_device: bad parameters")
        _raise(st)
        return rows[:ne], cols[:ne]
    rp = np.zeros(n + 1, np.int64)
    cap = max((2 if recipe == 1 else 1) * ne, 1)
    cl = np.zeros(cap, np.int64)
    vl = np.zeros(cap, np.float32) if recipe == 0 else None
    st = L.fmm_rmat_device(device, scale, edge_factor, *RMAT_ABC, seed, recipe, rp.ctypes.data_as(P64),
                           cl.ctypes.data_as(P64), None if vl is None else vl.ctypes.data_as(C.POINTER(C.c_float)),
                           None, None, C.byref(nnz))
    if st == _lib.FMM_E_INVAL:
        raise InvalidArgument("rmat_device: bad parameters")
    _raise(st)
    k = nnz.value
    return CsrMatrix(n, n, rp, cl[:k].copy(), None if vl is None else vl[:k].copy())


def rmat_stream(scale: int, edge_factor: int, seed: int):
    """Raw insertion stream (rows, cols) for cross-checks with the reference."""
    ne = edge_factor << scale
    rows = np.zeros(ne, np.int64)
    cols = np.zeros(ne, np.int64)
    _lib.gen().fmmgen_rmat_stream(scale, edge_factor, *RMAT_ABC, seed,
                                  rows.ctypes.data_as(C.POINTER(C.c_int64)),
                                  cols.ctypes.data_as(C.POINTER(C.c_int64)))
    return rows, cols


def normal_fill(count: int, scale: float, seed: int) -> np.ndarray:
    out = np.empty(count, np.float32)
    _lib.gen().fmmgen_normal_fill(out.ctypes.data_as(C.POINTER(C.c_float)), count, scale, seed)
    return out


def uniform_fill(count: int, lo: float, hi: float, seed: int) -> np.ndarray:
    out = np.empty(count, np.float32)
    _lib.gen().fmmgen_uniform_fill(out.ctypes.data_as(C.POINTER(C.c_float)), count, lo, hi, seed)
    return out


def config1(n: int = 16384, k: int = 16, d: int = 64, seed: int = 0) -> Workload:
    """ER digraph, exactly k distinct sorted out-neighbours per row, a_uv ~
    U(0,1), X ~ U(-1,1); GCN SpMM (SEL2ND, NOOP, NOOP, MUL, ASUM)."""
    rp = np.zeros(n + 1, np.int64)
    cl = np.zeros(n * k, np.int64)
    vl = np.zeros(n * k, np.float32)
    X = np.zeros(n * d, np.float32)
    P64 = C.POINTER(C.c_int64)
    PF = C.POINTER(C.c_float)
    rc = _lib.gen().fmmgen_er_fixed(n, k, seed, rp.ctypes.data_as(P64), cl.ctypes.data_as(P64),
                                    vl.ctypes.data_as(PF), X.ctypes.data_as(PF), d)
    if rc != 0:
        raise ValueError("config1: bad parameters")
    A = CsrMatrix(n, n, rp, cl, vl)
    return Workload("config1_gcn", A, DenseMatrix(n, d, X), make_spec(App.GCN_FORWARD), 1, True, True,
                    f"ER n={n} k={k} d={d} GCN SpMM, seed {seed}")


def _rmat_graph(scale: int, edge_factor: int, seed: int, gen: Optional[str]) -> CsrMatrix:
    """BASELINE R-MAT graph from the host builder ("host") or wholly on the
    GPU ("device", fmm_rmat_device); both are the same CSR (tested). The
    default follows FMM_GEN (host when unset)."""
    gen = gen or os.environ.get("FMM_GEN", "host")
    if gen == "device":
        return rmat_device(scale, edge_factor, seed, recipe=1)
    return rmat_sym(scale, edge_factor, seed)


def config2(scale: int = 20, edge_factor: int = 16, d: int = 128, seed: int = 1, gen: Optional[str] = None) -> Workload:
    """R-MAT sigmoid embedding; X ~ 0.1 N(0,1)."""
    A = _rmat_graph(scale, edge_factor, seed, gen)
    X = DenseMatrix.wrap(normal_fill(A.nrows * d, 0.1, seed).reshape(A.nrows, d))
    return Workload("config2_sigmoid", A, X, make_spec(App.NODE_EMBED_SIGMOID), 1, False, False,
                    f"R-MAT scale {scale} ef {edge_factor} d={d} sigmoid embedding, seed {seed}")


def config3(scale: int = 21, edge_factor: int = 8, d: int = 32, seed: int = 2, iters: int = 20,
            gen: Optional[str] = None) -> Workload:
    """R-MAT t-distribution layout; X ~ U(-10,10); 20 iterations X <- Z."""
    A = _rmat_graph(scale, edge_factor, seed, gen)
    X = DenseMatrix.wrap(uniform_fill(A.nrows * d, -10.0, 10.0, seed).reshape(A.nrows, d))
    return Workload("config3_tdist", A, X, tdist_spec(), iters, False, False,
                    f"R-MAT scale {scale} ef {edge_factor} d={d} t-distribution, {iters} iterations, seed {seed}")


def config4(side: int = 2048, seed: int = 3, k: float = 1.0) -> Workload:
    """2-D lattice + one random shortcut per vertex; X = lattice coords +
    0.01 N(0,1); FR-attractive |x_u-x_v|^2/k scaling the difference."""
    G = _lib.gen()
    n = side * side
    rp = C.POINTER(C.c_int64)()
    cl = C.POINTER(C.c_int64)()
    nnz = C.c_int64()
    X = np.zeros(n * 2, np.float32)
    rc = G.fmmgen_lattice(side, seed, C.byref(rp), C.byref(cl), C.byref(nnz),
                          X.ctypes.data_as(C.POINTER(C.c_float)))
    if rc != 0:
        raise ValueError("config4: bad parameters")
    A = CsrMatrix(n, n, _take(rp, n + 1, np.int64), _take(cl, nnz.value, np.int64), None)
    return Workload("config4_fr_attract", A, DenseMatrix.wrap(X.reshape(n, 2)), fr_attract_spec(k), 1,
                    False, True, f"{side}x{side} lattice + shortcut, d=2 FR-attractive k={k}, seed {seed}")


def config5(scale: int = 24, edge_factor: int = 32, d: int = 256, seed: int = 4, iters: int = 5,
            gen: Optional[str] = None) -> Workload:
    """Large R-MAT sigmoid embedding, 5 epochs X <- Z."""
    A = _rmat_graph(scale, edge_factor, seed, gen)
    X = DenseMatrix.wrap(normal_fill(A.nrows * d, 0.1, seed).reshape(A.nrows, d))
    return Workload("config5_sigmoid_large", A, X, make_spec(App.NODE_EMBED_SIGMOID), iters, False, False,
                    f"R-MAT scale {scale} ef {edge_factor} d={d} sigmoid, {iters} epochs, seed {seed}")


def get(config: int, small: bool = False) -> Workload:
    """Full-size config, or (small=True) the same recipe scaled for CPU parity."""
    if config == 1:
        return config1(n=2048) if small else config1()
    if config == 2:
        return config2(scale=13) if small else config2()
    if config == 3:
        return config3(scale=13, iters=3) if small else config3()
    if config == 4:
        return config4(side=128) if small else config4()
    if config == 5:
        return config5(scale=12, edge_factor=32, iters=2) if small else config5()
    raise ValueError(f"unknown config {config}")
