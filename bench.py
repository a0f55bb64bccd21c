#!/usr/bin/env python
"""FusedMM bench on B200 — one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Workload: BASELINE.json configs[1] (config 2: sigmoid graph embedding, R-MAT
scale 20, ef 16, d=128) by default; --config 3 / 5 select the iterative
workloads. Metric: nnz*d/s (whole job).

ours:      one step = one fused call over every rank's row block (part1d
           balanced on nnz plus a per-row cost; rows never split) with the
           inputs resident in HBM. For the iterative workloads (--config 3 /
           5) with N > 1 the step also carries the epoch's Z exchange: every
           finished z row is stored by the kernel itself, over NVLink (CUDA
           IPC), into the next-iterate buffer of each peer that reads it
           (halo masks), and a stream-ordered barrier closes the step; X is
           held fixed across steps, so every step moves the same bytes (an
           X <- Z feedback would move exactly these). Config 2 is one call:
           Z stays row-sharded, and the halo bytes an iteration would move
           are reported beside the line. Device time: CUDA events on the launch stream,
           max over ranks; L2 flushed (256 MiB write, then a 256 MiB read so no
           dirty lines are left) between timed steps
           outside the events. e2e: the same call through the C ABI with
           pinned HOST buffers (X host->device, Z device->host in the timed
           region). roofline: the row kernel's DRAM bytes per launch from the
           committed `ncu --set full` capture over the live launch time,
           against MEASURED_PEAKS.json; B_alg (every gather charged once)
           and the L2->SM delivery are reported beside it.
reference: the unmodified reference fusedmm::fused_mm<float> (oracle/_ref,
           compiled from /root/reference) on all host cores, its inputs built
           by the reference's own generator (oracle.ref_workload: rmat_generate
           + the BASELINE recipe; bitwise equal to ours, tests/test_oracle.py)
           — no library of this repo is loaded on that arm.
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


def ncu_capture(cfg: int):
    """(report dict, source) of the newest committed `ncu --set full` capture
    of this config's row kernel (profiles/<tag>_summary.json), or (None, why).
    Per launch: dram__bytes_read.sum + dram__bytes_write.sum, duration, L2->SM."""
    for path in sorted((ROOT / "profiles").glob("r*_summary.json"), reverse=True):
        try:
            s = json.loads(path.read_text())
        except Exception:
            continue
        for name, rep in s.get("reports", {}).items():
            if name.endswith(f"config{cfg}_rows") and "dram_bytes_total" in rep:
                return rep, f"{path.name}:{name} (ncu --set full, one launch)"
    return None, "no committed ncu capture for this config"


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


def config_dict(w) -> dict:
    """The `config` object of the JSON line: identical on both arms."""
    return {"workload": w.name, "desc": w.description, "rows": int(w.A.nrows), "nnz": int(w.A.nnz()),
            "d": int(w.d)}


# Workloads above this many edges are timed on the CPU through a row sample
# (config 5: ~1e9 edges, ~50-100 s per reference call).
CPU_SAMPLE_NNZ = 64_000_000


def cpu_sample(w, max_nnz: int = CPU_SAMPLE_NNZ):
    """(A_s, X_s, Y, description): the whole workload, or a seeded random
    subset of rows with about max_nnz edges (all columns kept, Y = full X).
    Plain oracle containers only (the reference arm loads no repo library)."""
    import oracle
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
    unit = bool(getattr(A, "unit_values", False))
    As = oracle._Csr(int(take.size), A.ncols, rp, A.col_idx[idx], None if unit else A.values[idx])
    Xs = oracle._Dense(np.ascontiguousarray(X.array[take]))
    return As, Xs, X, (f"{take.size} random rows of {w.name} ({As.nnz()} of {A.nnz()} edges), "
                       f"Y = full X")


def cpu_reference_run(w, steps: int, warmup: int, budget_s: float | None, threads: int | None = None):
    """Time the reference fused_mm<float> (oracle/_ref) or, when it was not
    built, the C restatement (oracle port) on all host threads (or
    `threads`). Returns the per-step seconds and the sample's nnz*d (the unit
    the rate counts)."""
    import oracle
    threads = threads or oracle.host_threads()
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
    """The reference's own CPU implementation on this box's host cores, on
    the same workload as ours (inputs from the reference generator when
    oracle/_ref is built: no library of this repo is loaded)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    t0 = time.time()
    if oracle.ref_available() and args.config in (2, 3, 5):
        w = oracle.ref_workload(args.config)
        inputs = "reference generator (oracle/_ref: rmat_generate + BASELINE recipe)"
    else:
        w, _ = load_workload(args.config)
        inputs = "repo host generator (libfmm_gen)"
    gen_s = time.time() - t0
    kind, threads, times, nnzd, sample = cpu_reference_run(w, args.steps, args.warmup, None)
    sec = sum(times) / len(times)
    value = nnzd / sec
    line = {
        "metric": "nnz*d/s", "impl": "reference", "value": value, "unit": "nnz*d/s",
        "n_gpus": world, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, BASELINE.json recipe)",
        "config": config_dict(w),
        "details": {"inputs": inputs, "gen_seconds": round(gen_s, 2)},
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
    from paper_2011_06391_b200.shard import ShardedFusedMM

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
    stream = torch.cuda.Stream(dev)  # the lib launches here; events are recorded here
    torch.cuda.set_stream(stream)

    # one rank's share: rows [rb, re) of the cost-balanced part1d partition
    sh = ShardedFusedMM(A, d, spec, device=dev, exchange="fused")
    sh.ctx.set_stream(0, stream.cuda_stream)
    rb, re = sh.rb, sh.re
    g = sh.graph
    info = g.info()

    X_dev = torch.from_numpy(X.array).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    # FMM_BENCH_FLUSH=write+read: the write pass is followed by a read pass over
    # a second 256 MiB buffer, so the step starts on a cold L2 without ~126 MB
    # of dirty flush lines to write back during the timed kernel
    flush_mode = os.environ.get("FMM_BENCH_FLUSH", "write+read")
    flush_rd = torch.zeros(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if flush_mode == "write+read" else None
    flush_acc = torch.zeros(1, dtype=torch.float32, device=dev)

    def flush_l2():
        flush.zero_()
        if flush_rd is not None:
            torch.sum(flush_rd, dim=0, keepdim=True, out=flush_acc)
    st = _lib.fmm_stats()
    exchange = None
    iterative = w.iters > 1  # configs 3 and 5: X <- Z between iterations / epochs
    if world > 1:
        sh.set_halo_masks()
    if world > 1 and not iterative:
        # config 2 is ONE fused call (BASELINE.json): each rank writes its row
        # block of Z, as the reference's workers write disjoint row ranges of
        # one Z (kernel.hpp:335-345); no exchange belongs to the call. The
        # halo bytes an iterated embedding would move are reported beside it.
        Z_dev = torch.empty((re - rb, d), dtype=torch.float32, device=dev)

        def step():
            g.run_device(X_dev.data_ptr(), m, X_dev.data_ptr(), Z_dev.data_ptr(), d, spec, stats=st)
        sent = torch.tensor([sh.exchange_rows * d * 4, sh.exchange_rows_all * d * 4], dtype=torch.float64,
                            device=dev)
        tot = sent.clone()
        dist.all_reduce(tot)
        exchange = {"in_step": False,
                    "why": "single-call workload: Z stays row-sharded (no collective on the data path)",
                    "halo_bytes_per_iteration_if_iterated": int(tot[0].item()),
                    "all_rows_bytes_per_iteration": int(tot[1].item())}
    elif world > 1:
        # the epoch's Z exchange, fused into the kernel: z rows go straight
        # into each reading peer's next-iterate buffer (halo masks)
        nxt = torch.empty_like(X_dev)
        peers = sh.map_peer_buffers([nxt])
        peer_next = [peers[q][0] for q in sorted(peers)]

        def step():
            sh.step_exchange(X_dev, nxt, peer_next)
        sent = torch.tensor([sh.exchange_rows * d * 4, sh.exchange_rows_all * d * 4], dtype=torch.float64,
                            device=dev)
        tot = sent.clone()
        dist.all_reduce(tot)
        mx = sent.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        barrier = "a host barrier (gloo, ranks sharing one GPU: test mode)" if share else \
            "a stream-ordered NCCL barrier"
        exchange = {"in_step": True,
                    "how": "in-kernel P2P stores (CUDA IPC over NVLink) of each z row into the next-iterate "
                           f"buffer of every peer that reads it, then {barrier}",
                    "bytes_per_step_total": int(tot[0].item()), "bytes_per_step_max_rank": int(mx[0].item()),
                    "bytes_per_step_without_halo_masks": int(tot[1].item()),
                    "cut_by_masks": 1.0 - float(tot[0].item()) / max(float(tot[1].item()), 1.0)}
    else:
        Z_dev = torch.empty((re - rb, d), dtype=torch.float32, device=dev)

        def step():
            g.run_device(X_dev.data_ptr(), m, X_dev.data_ptr(), Z_dev.data_ptr(), d, spec, stats=st)

    launches0 = sh.launches
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = ((sh.launches - launches0) // max(args.warmup, 1) if (world > 1 and iterative)
                         else int(st.launches))

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
        flush_l2()
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
    mean_ms = kernel_ms_total / args.steps

    # ---- roofline of the row kernel: DRAM bytes per launch (committed ncu
    # capture of the same kernel on the whole graph) over the live launch time
    nnz_r = int(A.row_ptr[re] - A.row_ptr[rb])
    rows_r = re - rb
    deg = np.diff(A.row_ptr[rb:re + 1])
    # compulsory (each array once): row_ptr, columns, values, X, Z
    compulsory = (8 * (rows_r + 1) + 4 * nnz_r + (4 * nnz_r if w.weighted else 0)
                  + 4 * d * A.ncols + 4 * d * rows_r)
    b_alg = (8 * (rows_r + 1) + 4 * nnz_r + 4 * d * nnz_r + 4 * d * rows_r
             + (4 * nnz_r if w.weighted else 0) + (4 * d * int(np.count_nonzero(deg)) if spec.vop != 2 else 0))
    peak, peak_src = hbm_peak()
    cap, cap_src = ncu_capture(args.config)
    roofline = {"bound": "hbm", "peak": peak, "unit": "GB/s", "peak_source": peak_src,
                "kernel": "fmm_rows_kernel (split-row chunks folded in-kernel)"}
    if cap is not None and world == 1:
        traffic = float(cap["dram_bytes_total"])
        achieved = traffic / (mean_ms / 1e3) / 1e9
        roofline.update({
            "achieved": achieved, "frac": achieved / peak, "traffic": traffic, "traffic_source": cap_src,
            "what": "achieved = ncu DRAM bytes (read + write) per launch / live mean launch time",
            "ncu_kernel": cap.get("kernel"), "ncu_launch_ms": 1e3 * float(cap["gpu__time_duration.sum"]),
            "ncu_dram_throughput_pct": cap.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")})
        l2b = cap.get("l1tex__m_xbar2l1tex_read_bytes.sum")
        if l2b is not None:
            roofline["l2_to_sm"] = {"bytes_per_launch": float(l2b),
                                    "achieved_gbs": float(l2b) / (mean_ms / 1e3) / 1e9,
                                    "what": "L2->SM bytes (ncu l1tex__m_xbar2l1tex_read_bytes) / launch time"}
    else:
        roofline.update({"achieved": None, "frac": None, "traffic": None,
                         "traffic_source": cap_src if cap is None else "per-rank shard: whole-graph capture n/a"})
    roofline["compulsory_bytes"] = compulsory
    roofline["compulsory_frac"] = compulsory / (mean_ms / 1e3) / 1e9 / peak
    roofline["gather_bytes"] = b_alg
    roofline["gather_bytes_what"] = ("B_alg of SURVEY.md 8(d): every y_v gather charged once (most are "
                                     "served by L2, so B_alg/t is not an HBM rate)")

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
        # the reference's single-thread rate beside it
        _, _, t1, nnzd_1, _ = cpu_reference_run(w, 1, 0, budget_s=None, threads=1)
        cpu["value_1_thread"] = nnzd_1 / t1[0]

    if world > 1 and iterative:
        sh.unmap_peer_buffers()
    g_e.free()
    ctx_e.close()
    sh.close()
    Xh.close()
    Zh.close()
    if rank == 0:
        line = {
            "metric": "nnz*d/s", "value": value, "unit": "nnz*d/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded, BASELINE.json recipe)",
            "config": config_dict(w),
            "details": {"parallelism": f"row-shard x{world} (part1d, nnz + per-row cost)",
                        "l2": ("flushed between timed steps (256 MiB write then 256 MiB read: cold and clean, outside the events)"
                               if flush_mode == "write+read" else
                               "flushed between timed steps (256 MiB write, outside the events)"),
                        "split_rows": int(info.split_rows), "max_degree": int(info.max_degree),
                        "gen_seconds": round(gen_s, 2),
                        "step": ("fused call + halo exchange of the epoch's Z (X fixed across steps)"
                                 if (world > 1 and iterative) else "one fused call")},
            "exchange": exchange,
            "roofline": roofline,
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
    ap.add_argument("--steps", type=int, default=50)
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
