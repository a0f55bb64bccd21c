#!/usr/bin/env python
"""FusedMM bench on B200 — one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Workload: BASELINE.json configs[1] (config 2: sigmoid graph embedding, R-MAT
scale 20, ef 16, d=128), one fused call per step. Metric: nnz*d/s (whole job)
with the achieved HBM roofline fraction of the fused kernel alongside.

ours:      inputs resident in HBM, kernel timed with CUDA events on the launch
           stream, L2 flushed (256 MiB write) between timed steps outside the
           events; rows split across ranks by part1d balanced on nnz plus a
           per-row cost (fmm_part1d_weighted; strong scaling:
           the graph is fixed, each rank computes its row block).
           e2e: the same call through the C ABI with pinned HOST buffers
           (X host->device, Z device->host inside the timed region).
reference: the unmodified reference fusedmm::fused_mm<float> (oracle/_ref,
           compiled from /root/reference) on the host cores, all threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0


def ncu_traffic(cfg: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the row
    kernel for this config, from the newest committed `ncu --set full`
    capture (profiles/<tag>_summary.json), or (None, why)."""
    for path in sorted((ROOT / "profiles").glob("r*_summary.json"), reverse=True):
        try:
            s = json.loads(path.read_text())
        except Exception:
            continue
        for name, rep in s.get("reports", {}).items():
            if name.endswith(f"config{cfg}_rows") and "dram_bytes_total" in rep:
                return rep["dram_bytes_total"], f"{path.name}:{name} (ncu --set full, one launch)"
    return None, "no committed ncu capture for this config"


def l2_delivery(cfg: int):
    """(L2->SM bytes per launch of the row kernel from the newest committed
    ncu capture, the measured delivery ceiling of config 2's own gather
    stream (tools/gather_pattern.py: plain row gathers of the real CSR column
    stream, best shape), source) or Nones."""
    got, src = None, None
    for path in sorted((ROOT / "profiles").glob("r*_summary.json"), reverse=True):
        try:
            s = json.loads(path.read_text())
        except Exception:
            continue
        for name, rep in s.get("reports", {}).items():
            if name.endswith(f"config{cfg}_rows") and "l1tex__m_xbar2l1tex_read_bytes.sum" in rep:
                got, src = rep["l1tex__m_xbar2l1tex_read_bytes.sum"], f"{path.name}:{name}"
                break
        if got is not None:
            break
    ceiling = None
    if cfg == 2:
        for path in sorted((ROOT / "profiles").glob("r*_gather_pattern.log"), reverse=True):
            vals = [float(l.split()[-2]) for l in path.read_text().splitlines()
                    if (l.startswith("/tmp/g_csr.bin") or l.startswith("/tmp/g2_csr.bin")) and l.endswith("TB/s")]
            if vals:
                ceiling = (max(vals) * 1e3, path.name)
                break
    return got, src, ceiling


def hbm_peak():
    try:
        p = json.loads(PEAKS_FILE.read_text())
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_workload(cfg: int):
    from paper_2011_06391_b200 import configs
    t0 = time.time()
    w = configs.get(cfg, small=False)
    return w, time.time() - t0


# Workloads above this many edges are timed on the CPU through a row sample
# (config 5: ~1e9 edges, ~50-100 s per reference call).
CPU_SAMPLE_NNZ = 64_000_000


def cpu_sample(w, max_nnz: int = CPU_SAMPLE_NNZ):
    """(A_s, X_s, Y, description): the whole workload, or a seeded random
    subset of rows with about max_nnz edges (all columns kept, Y = full X)."""
    from paper_2011_06391_b200 import fusedmm as F
    A, X = w.A, w.X
    if A.nnz() <= max_nnz:
        return A, X, X, f"full {w.name} fused_mm call"
    rng = np.random.default_rng(12345)
    deg = np.diff(A.row_ptr)
    perm = rng.permutation(A.nrows)
    take = np.sort(perm[:int(np.searchsorted(np.cumsum(deg[perm]), max_nnz)) + 1])
    rp = np.concatenate([[0], np.cumsum(deg[take])]).astype(np.int64)
    idx = np.concatenate([np.arange(A.row_ptr[r], A.row_ptr[r + 1]) for r in take]) if take.size else \
        np.zeros(0, np.int64)
    As = F.CsrMatrix(int(take.size), A.ncols, rp, A.col_idx[idx], None if A.unit_values else A.values[idx])
    Xs = F.DenseMatrix.wrap(X.array[take])
    return As, Xs, X, (f"{take.size} random rows of {w.name} ({As.nnz()} of {A.nnz()} edges), "
                       f"Y = full X")


def cpu_reference_run(w, steps: int, warmup: int, budget_s: float | None):
    """Time the reference fused_mm<float> (oracle/_ref) or, when it was not
    built, the C restatement (oracle port) on all host threads. Returns the
    per-step seconds and the sample's nnz*d (the unit the rate counts)."""
    import oracle
    threads = oracle.host_threads()
    As, Xs, Y, sample = cpu_sample(w)
    if oracle.ref_available():
        call = oracle.RefCall(As, Xs, Y, w.spec)
        kind = "reference"

        def one():
            return call.run(threads, want_z=False)[1]
    else:
        kind = "port"

        def one():
            t0 = time.perf_counter()
            oracle.oracle_fused_mm(As, Xs, Y, w.spec, threads=threads)
            return time.perf_counter() - t0
    for _ in range(warmup):
        one()
    times = []
    t_start = time.perf_counter()
    for _ in range(steps):
        times.append(one())
        if budget_s is not None and time.perf_counter() - t_start > budget_s:
            break
    return kind, threads, times, As.nnz() * w.d, sample


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    w, _ = load_workload(args.config)
    kind, threads, times, nnzd, sample = cpu_reference_run(w, args.steps, args.warmup, None)
    sec = sum(times) / len(times)
    value = nnzd / sec
    line = {
        "metric": "nnz*d/s", "impl": "reference", "value": value, "unit": "nnz*d/s",
        "n_gpus": world, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, BASELINE.json recipe)",
        "config": {"workload": w.name, "desc": w.description, "nnz": w.A.nnz(), "d": w.d,
                   "rows": w.A.nrows},
        "cpu_baseline": {"value": value, "unit": "nnz*d/s", "cores": threads, "kind": kind,
                         "sample": f"{sample} per step ({len(times)} steps)"},
        "e2e": {"value": value, "unit": "nnz*d/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2011_06391_b200 import fusedmm as F
    from paper_2011_06391_b200 import _lib

    rank, world, local = dist_env()
    # FMM_BENCH_SHARE_GPU=1 (testing only): every rank on GPU 0 with gloo, to
    # exercise the multi-rank code path on a one-GPU box (timings meaningless)
    share = os.environ.get("FMM_BENCH_SHARE_GPU") == "1"
    if world > 1:
        torch.cuda.set_device(0 if share else local)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    w, gen_s = load_workload(args.config)
    A, X, spec, d = w.A, w.X, w.spec, w.d
    m = A.nrows
    plan = F.shard_bounds(A, world, d)  # part1d balanced on nnz + per-row cost
    rb, re = plan.boundaries[rank], plan.boundaries[rank + 1]

    ctx = F.Context([dev.index])
    stream = torch.cuda.Stream(dev)  # the lib launches here; events are recorded here
    torch.cuda.set_stream(stream)
    ctx.set_stream(0, stream.cuda_stream)
    g = F.DeviceGraph(ctx, A, rb, re)
    info = g.info()

    X_dev = torch.from_numpy(X.array).to(dev)
    Z_dev = torch.empty((re - rb, d), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    st = _lib.fmm_stats()

    def step():
        g.run_device(X_dev.data_ptr(), m, X_dev.data_ptr(), Z_dev.data_ptr(), d, spec, stats=st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = int(st.launches)

    # ---- timed region: K steps, L2 flushed between steps outside the events
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    clocks = ClockSampler(dev.index)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    kernel_ms_total = sum(step_ms)
    t_rank = torch.tensor([kernel_ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_rank, op=dist.ReduceOp.MAX)
    t_max_ms = float(t_rank.item())

    nnzd_total = A.nnz() * d
    value = nnzd_total * args.steps / (t_max_ms / 1e3)

    # roofline of this rank's fused kernels: algorithmic bytes per launch
    nnz_r = int(A.row_ptr[re] - A.row_ptr[rb])
    rows_r = re - rb
    deg = np.diff(A.row_ptr[rb:re + 1])
    alg = (8 * (rows_r + 1) + 4 * nnz_r + 4 * d * nnz_r + 4 * d * rows_r
           + (4 * nnz_r if w.weighted else 0) + (4 * d * int(np.count_nonzero(deg)) if spec.vop != 2 else 0))
    mean_ms = kernel_ms_total / args.steps
    achieved = alg / (mean_ms / 1e3) / 1e9
    peak, peak_src = hbm_peak()
    l2_bytes, l2_src, l2_ceiling = l2_delivery(args.config)
    delivery = None
    if l2_bytes is not None:
        ach = l2_bytes * (nnz_r / max(A.nnz(), 1)) / (mean_ms / 1e3) / 1e9
        delivery = {"what": "L2->SM bytes of the row kernel (ncu l1tex__m_xbar2l1tex_read_bytes) per launch time",
                    "achieved": ach, "unit": "GB/s", "bytes_source": l2_src,
                    "ceiling": l2_ceiling[0] if l2_ceiling else None,
                    "frac": ach / l2_ceiling[0] if l2_ceiling else None,
                    "ceiling_source": (f"{l2_ceiling[1]}: plain row gathers of this config's CSR column "
                                       "stream, best load width / occupancy") if l2_ceiling else None}

    # ---- e2e through the C ABI with pinned host buffers
    Xh = F.PinnedBuffer(X.array.shape)  # fmm_host_alloc: page-locked
    Xh.array[:] = X.array
    Zh = F.PinnedBuffer((rows_r, d))
    Xh_np, Zh_np = Xh.array, Zh.array
    ctx_e = F.Context([dev.index])
    g_e = F.DeviceGraph(ctx_e, A, rb, re)
    e2e_steps = max(3, min(args.steps, 50 if m * d * 4 < (4 << 30) else 3))

    def e2e_run(flags: int) -> float:
        for _ in range(max(1, args.warmup)):
            g_e.run_host(Xh_np, Xh_np, Zh_np, d, spec, flags)
        ctx_e.sync()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            g_e.run_host(Xh_np, Xh_np, Zh_np, d, spec, flags)
        ctx_e.sync()  # every step's Z is back in host memory
        t_e = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        return nnzd_total * e2e_steps / float(t_e.item())

    # synchronous calls (fused_mm semantics), then the pipelined FMM_ASYNC
    # host path: upload of step k+1 overlaps download of step k (full duplex)
    e2e_sync = e2e_run(0)
    e2e_value = e2e_run(_lib.FMM_ASYNC)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        kind, threads, times, nnzd_s, sample = cpu_reference_run(w, 20, 1, budget_s=20.0)
        sec = sum(times) / len(times)
        cpu = {"value": nnzd_s / sec, "unit": "nnz*d/s", "cores": threads, "kind": kind,
               "sample": f"{sample} x{len(times)} (1 warm-up), all host threads"}

    if rank == 0:
        line = {
            "metric": "nnz*d/s", "value": value, "unit": "nnz*d/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded, BASELINE.json recipe)",
            "config": {"workload": w.name, "desc": w.description, "rows": m, "nnz": A.nnz(), "d": d,
                       "parallelism": f"row-shard x{world} (part1d, nnz + per-row cost)",
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "split_rows": int(info.split_rows), "max_degree": int(info.max_degree),
                       "gen_seconds": round(gen_s, 2)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(args.config)[0],
                         "traffic_source": ncu_traffic(args.config)[1],
                         "alg_bytes_per_launch": alg, "peak_source": peak_src,
                         "kernel": "fmm_rows_kernel (split-row chunks folded in-kernel)",
                         "l2_to_sm": delivery},
            "e2e": {"value": e2e_value, "unit": "nnz*d/s", "h2d_bytes_per_step": int(m * d * 4),
                    "d2h_bytes_per_step": int(rows_r * d * 4), "steps": e2e_steps,
                    "how": "fmm_run(FMM_HOST_PTRS|FMM_ASYNC) pinned host X in / Z out every step, fmm_sync",
                    "sync_calls_value": e2e_sync},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk, "wall_s_timed_region": wall,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
