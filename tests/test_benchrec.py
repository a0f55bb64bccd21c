"""BenchRecord / write_csv / run_bench on the device (bench.hpp:21-190,
perf.hpp:21-32): the CSV is byte-identical to the reference's writer (pinned
through oracle/_ref) and the reference's own bench tests
(proj/tests/test_io.cpp:145-199) hold on the device."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2011_06391_b200 import benchrec as B
from paper_2011_06391_b200 import fusedmm as F

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


class RefRecord(C.Structure):
    _fields_ = [("graph", C.c_char_p), ("app", C.c_char_p), ("m", C.c_int64), ("n", C.c_int64),
                ("nnz", C.c_int64), ("d", C.c_int64), ("avg_degree", C.c_double), ("threads", C.c_int32),
                ("iterations", C.c_int32), ("fused_seconds", C.c_double), ("reference_seconds", C.c_double),
                ("speedup", C.c_double), ("achieved_gflops", C.c_double), ("ai_lower_bound", C.c_double),
                ("fused_aux_bytes", C.c_uint64), ("materialized_h_bytes", C.c_uint64),
                ("reference_oom", C.c_int32), ("verified", C.c_int32)]


def _records():
    rng = np.random.default_rng(3)
    out = [B.BenchRecord(), B.BenchRecord(graph="with,comma", app='q"uote'),
           B.BenchRecord(graph="rmat20", m=1048576, n=1048576, nnz=31398704, avg_degree=29.943771362304688,
                         d=128, app="embed", threads=8, iterations=10, fused_seconds=0.0012061,
                         reference_seconds=0.00386, speedup=3.2004, achieved_gflops=13327.5,
                         ai_lower_bound=0.9084, fused_aux_bytes=1 << 30, materialized_h_bytes=125594816,
                         reference_oom=False, verified=False)]
    for i in range(6):
        out.append(B.BenchRecord(graph=f"g{i}\nline", m=int(rng.integers(1, 1 << 40)), n=3, nnz=5,
                                 avg_degree=float(rng.uniform(0, 1e6)), d=int(rng.integers(1, 4096)),
                                 app="fr", threads=i, iterations=i * 3,
                                 fused_seconds=float(10.0 ** rng.uniform(-9, 3)),
                                 reference_seconds=float(rng.uniform(0, 1e-4)),
                                 speedup=float(rng.uniform(0, 1e7)), achieved_gflops=1e-300 * i,
                                 ai_lower_bound=float(rng.uniform()), reference_oom=bool(i % 2),
                                 verified=bool(i % 3)))
    return out


def test_write_csv_shapes():
    """test_io.cpp:145-159."""
    assert B.csv_string([]).count("\n") == 1
    body = B.csv_string([B.BenchRecord(graph="plain"), B.BenchRecord(graph="with,comma")])
    assert body.count("\n") == 3 and '"with,comma"' in body


@needs_ref
def test_write_csv_bytes_equal_reference(tmp_path):
    recs = _records()
    L = oracle.ref_lib()
    L.fmm_ref_write_csv.argtypes = [C.c_char_p, C.c_int, C.POINTER(RefRecord)]
    arr = (RefRecord * len(recs))()
    for a, r in zip(arr, recs):
        a.graph, a.app = r.graph.encode(), r.app.encode()
        for f in ("m", "n", "nnz", "d", "avg_degree", "threads", "iterations", "fused_seconds",
                  "reference_seconds", "speedup", "achieved_gflops", "ai_lower_bound", "fused_aux_bytes",
                  "materialized_h_bytes"):
            setattr(a, f, getattr(r, f))
        a.reference_oom, a.verified = int(r.reference_oom), int(r.verified)
    assert L.fmm_ref_write_csv(str(tmp_path / "ref.csv").encode(), len(recs), arr) == 0
    B.write_csv(recs, tmp_path / "ours.csv")
    assert (tmp_path / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()


@needs_ref
@pytest.mark.parametrize("deg,d", [(1.0, 1), (29.94, 128), (61.0, 256), (3.5, 7)])
def test_arithmetic_intensity_matches_reference(deg, d):
    L = oracle.ref_lib()
    L.fmm_ref_arithmetic_intensity.restype = C.c_double
    L.fmm_ref_arithmetic_intensity.argtypes = [C.c_double, C.c_int64]
    assert B.arithmetic_intensity(deg, d) == L.fmm_ref_arithmetic_intensity(deg, d)
    assert B.flop_count(31398704, d) == 4 * d * 31398704
    with pytest.raises(F.InvalidArgument):
        B.arithmetic_intensity(0.0, d)


def _rmat(scale, ef, seed):
    rp, cl, vl = oracle.ref_rmat(scale, ef, seed)
    return F.CsrMatrix(1 << scale, 1 << scale, rp, cl, vl)


@pytest.mark.gpu
def test_run_bench_smoke_on_device():
    """test_io.cpp:161-180, t = GPU shards {1, 2} (shards share GPU 0 here)."""
    A = _rmat(8, 8, 11)
    recs = B.run_bench(A, "smoke", F.make_spec(F.App.NODE_EMBED_SIGMOID), "embed", [32], [1, 2], 2, B.BenchMode.BOTH)
    assert len(recs) == 2
    r1 = recs[0]
    assert r1.fused_seconds > 0 and r1.reference_seconds > 0 and r1.verified and not r1.reference_oom
    assert r1.achieved_gflops > 0 and r1.iterations == 2 and r1.speedup > 0
    assert recs[1].fused_seconds > 0 and recs[1].reference_oom  # unfused pipeline: one shard only
    assert B.csv_string(recs).count("\n") == 3


@pytest.mark.gpu
def test_run_bench_materialized_bytes_grow_with_d():
    """test_io.cpp:183-199 on the device with a vector-message spec (the
    device pipeline keeps one scalar per edge for scalar messages such as
    FR's, so its growth with d shows on vector messages): nnz*d message
    values (4 B each here) plus the edge-id gather index."""
    A = _rmat(8, 8, 13)
    spec = F.OpSpec(F.Vop.ADD, F.Rop.NOOP, F.Sop.SIGMOID, F.Mop.MUL, F.Aop.ASUM)
    recs = B.run_bench(A, "vec-growth", spec, "vec", [32, 64, 128], [1], 1, B.BenchMode.REFERENCE)
    assert len(recs) == 3
    sizes = [r.materialized_h_bytes for r in recs]
    assert sizes[0] < sizes[1] < sizes[2]
    for r in recs:
        assert r.materialized_h_bytes >= A.nnz() * r.d * 4
        assert r.fused_seconds == 0.0 and r.reference_seconds > 0
