"""Multi-GPU row sharding: one process per GPU over torch.distributed.

The reference's only parallelism is t std::thread workers over part1d row
ranges with X/Z partitioned and Y shared read-only (kernel.hpp:290-345,
PAPER.md:480-496). Here each rank is one GPU: rank r owns rows
[b_r, b_{r+1}) of part1d(A, world) balanced on nnz plus a per-row cost
(fmm_part1d_weighted), holds X (= Y) replicated in HBM and
computes its Z slice with the fused kernel — no collective on the data path.
Iterative workloads (configs 3 and 5: X <- Z) exchange the fresh Z slices
between iterations. Default on GPUs ("fused"): the ranks map each other's
X buffers once (CUDA IPC) and the fused kernel itself stores every finished
z row into its own next-X buffer and into every peer's (fmm_run_peers, P2P
stores over NVLink), so the all-gather overlaps the compute row by row; one
barrier per iteration (a stream-ordered NCCL all-reduce of one element, or a
host barrier under gloo) orders the next iteration after every rank's
kernel. "broadcast": every rank broadcasts its slice into every peer's
next-X buffer after the kernel (NCCL / gloo). Slices are unequal
(nnz-balanced, not row-balanced), so that is one broadcast per root rather
than a padded all-gather. Because rows are never split across ranks
and chunk boundaries are row-relative, results are bitwise independent of
the rank count.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist

from .fusedmm import CsrMatrix, Context, DeviceGraph, OpSpec, shard_bounds

# compute(X_full, Y_full, row_begin, row_end) -> Z slice (row_end-row_begin, d)
ComputeFn = Callable[[torch.Tensor, torch.Tensor, int, int], torch.Tensor]


class ShardedFusedMM:
    def __init__(self, A: CsrMatrix, d: int, spec: OpSpec, group=None,
                 device: Optional[torch.device] = None, compute: Optional[ComputeFn] = None,
                 exchange: str = "fused"):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.A, self.d, self.spec = A, d, spec
        # cost-balanced part1d (nnz + w(d) per row): rows are never split, so
        # the result is bitwise independent of the partition
        self.bounds = shard_bounds(A, self.world, d).boundaries
        self.rb, self.re = self.bounds[self.rank], self.bounds[self.rank + 1]
        self.launches = 0
        if exchange not in ("fused", "broadcast"):
            raise ValueError("exchange must be 'fused' or 'broadcast'")
        self.exchange_mode = exchange if (compute is None and self.world > 1) else "broadcast"
        if compute is not None:
            self._compute = compute
            self.device = device or torch.device("cpu")
        else:
            self.device = device or torch.device("cuda", torch.cuda.current_device())
            self.ctx = Context([self.device.index])
            self.ctx.set_stream(0, torch.cuda.current_stream(self.device).cuda_stream)
            self.graph = DeviceGraph(self.ctx, A, self.rb, self.re)
            self._compute = self._device_compute

    def _device_compute(self, X: torch.Tensor, Y: torch.Tensor, rb: int, re: int,
                        out: Optional[torch.Tensor] = None) -> torch.Tensor:
        Z = out if out is not None else torch.empty((re - rb, self.d), dtype=torch.float32,
                                                     device=self.device)
        from ._lib import fmm_stats
        st = fmm_stats()
        self.graph.run_device(X.data_ptr(), Y.shape[0], Y.data_ptr(), Z.data_ptr(), self.d,
                              self.spec, stats=st)
        self.launches += st.launches
        return Z

    def step(self, X: torch.Tensor, Y: Optional[torch.Tensor] = None) -> torch.Tensor:
        """This rank's Z slice for one fused call (no collective)."""
        Y = X if Y is None else Y
        return self._compute(X, Y, self.rb, self.re)

    def exchange(self, X_next: torch.Tensor) -> None:
        """Every rank's rows [b_r, b_{r+1}) of X_next are broadcast from rank r
        (in place, grouped, one root per slice)."""
        if self.world == 1:
            return
        works = []
        for r in range(self.world):
            b, e = self.bounds[r], self.bounds[r + 1]
            if e > b:
                works.append(dist.broadcast(X_next[b:e], src=r, group=self.group, async_op=True))
        for wk in works:
            wk.wait()

    def _barrier(self) -> None:
        """Orders the next iteration after every rank's kernel."""
        if dist.get_backend(self.group) == "nccl":
            flag = torch.zeros(1, device=self.device)
            dist.all_reduce(flag, group=self.group)  # stream-ordered: waits for every rank's kernel
        else:
            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.group)

    def _iterate_fused(self, X0: torch.Tensor, iters: int) -> torch.Tensor:
        from . import fusedmm as F
        from ._lib import fmm_stats
        bufs = [X0.clone(), torch.empty_like(X0)]
        torch.cuda.synchronize(self.device)
        mine = [F.ipc_handle(b.data_ptr()) for b in bufs]
        every: list = [None] * self.world
        dist.all_gather_object(every, mine, group=self.group)
        dev = self.device.index
        # (mapped base, offset) per peer buffer; the mapping is unmapped by base
        maps: dict = {}
        row_off = self.rb * self.d * 4
        try:
            # both buffers of a peer may live in one caching-allocator
            # segment (the same handle): map each distinct handle once
            for q in range(self.world):
                if q != self.rank:
                    maps[q] = {}
                    for (h, _off) in every[q]:
                        if h not in maps[q]:
                            maps[q][h] = F.ipc_open(h, dev)
            peers = {q: [maps[q][h] + off for (h, off) in every[q]] for q in maps}
            self._barrier()
            for it in range(iters):
                cur, nxt = bufs[it % 2], bufs[(it + 1) % 2]
                targets = [peers[q][(it + 1) % 2] + row_off for q in sorted(peers)]
                st = fmm_stats()
                self.graph.run_device_peers(cur.data_ptr(), cur.shape[0], cur.data_ptr(),
                                            nxt[self.rb:self.re].data_ptr(), self.d, self.spec, targets,
                                            stats=st)
                self.launches += st.launches
                self._barrier()  # every slice landed everywhere; nobody still reads `cur`
            out = bufs[iters % 2]
            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.group)  # no rank unmaps while a peer may still store into it
        finally:
            for q in maps:
                for base in maps[q].values():
                    F.ipc_close(base)
        return out

    def iterate(self, X0: torch.Tensor, iters: int) -> torch.Tensor:
        """iters fused calls with X <- Z; returns the replicated final X."""
        if self.exchange_mode == "fused":
            return self._iterate_fused(X0, iters)
        cur = X0.clone()
        nxt = torch.empty_like(cur)
        for _ in range(iters):
            if self._compute is self._device_compute:
                self._device_compute(cur, cur, self.rb, self.re, out=nxt[self.rb:self.re])
            else:
                nxt[self.rb:self.re] = self._compute(cur, cur, self.rb, self.re)
            self.exchange(nxt)
            cur, nxt = nxt, cur
        return cur
