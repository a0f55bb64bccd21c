"""Multi-GPU row sharding: one process per GPU over torch.distributed.

The reference's only parallelism is t std::thread workers over part1d row
ranges with X/Z partitioned and Y shared read-only (kernel.hpp:290-345,
PAPER.md:480-496). Here each rank is one GPU: rank r owns rows
[b_r, b_{r+1}) of part1d(A, world), holds X (= Y) replicated in HBM and
computes its Z slice with the fused kernel — no collective on the data path.
Iterative workloads (configs 3 and 5: X <- Z) exchange the fresh Z slices
between iterations: every rank broadcasts its slice into every peer's next-X
buffer (NCCL over NVLink on GPUs, gloo in the CPU tests). Slices are unequal
(nnz-balanced, not row-balanced), so the exchange is one broadcast per root
rather than a padded all-gather. Because rows are never split across ranks
and chunk boundaries are row-relative, results are bitwise independent of
the rank count.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist

from .fusedmm import CsrMatrix, Context, DeviceGraph, OpSpec, part1d

# compute(X_full, Y_full, row_begin, row_end) -> Z slice (row_end-row_begin, d)
ComputeFn = Callable[[torch.Tensor, torch.Tensor, int, int], torch.Tensor]


class ShardedFusedMM:
    def __init__(self, A: CsrMatrix, d: int, spec: OpSpec, group=None,
                 device: Optional[torch.device] = None, compute: Optional[ComputeFn] = None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.A, self.d, self.spec = A, d, spec
        self.bounds = part1d(A, self.world).boundaries
        self.rb, self.re = self.bounds[self.rank], self.bounds[self.rank + 1]
        self.launches = 0
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

    def iterate(self, X0: torch.Tensor, iters: int) -> torch.Tensor:
        """iters fused calls with X <- Z; returns the replicated final X."""
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
