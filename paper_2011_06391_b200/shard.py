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
                 exchange: str = "fused", halo: bool = True):
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
        self.halo = halo
        # rows this rank stores into peers per exchange (fused mode, after
        # the halo masks are set) and the unmasked count, for reporting
        self.exchange_rows = (self.re - self.rb) * (self.world - 1)
        self.exchange_rows_all = self.exchange_rows
        self._user_compute = compute  # None: the device path (no bound method kept: no cycle)
        self.ctx = None
        self.graph = None
        self._masks_set = False
        if compute is not None:
            self.device = device or torch.device("cpu")
        else:
            self.device = device or torch.device("cuda", torch.cuda.current_device())
            self.ctx = Context([self.device.index])
            self.ctx.set_stream(0, torch.cuda.current_stream(self.device).cuda_stream)
            self.graph = DeviceGraph(self.ctx, A, self.rb, self.re)

    def close(self) -> None:
        """Release the device graph and context now (do not leave it to
        finalisers at interpreter exit)."""
        if self.graph is not None:
            self.graph.free()
            self.graph = None
        if self.ctx is not None:
            self.ctx.close()
            self.ctx = None

    def __enter__(self) -> "ShardedFusedMM":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    def _compute(self, X: torch.Tensor, Y: torch.Tensor, rb: int, re: int,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if self._user_compute is not None:
            Z = self._user_compute(X, Y, rb, re)
            if out is not None:
                out.copy_(Z)
                return out
            return Z
        return self._device_compute(X, Y, rb, re, out)

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

    def set_halo_masks(self) -> None:
        """Per-row peer masks for the fused exchange: every rank publishes
        which rows its edges read (fmm_graph_column_use, n bytes), and this
        rank stores row r only to the peers that read it. Rows nobody else
        reads — every empty row of a symmetric graph, and rows referenced
        only from inside this block — are never sent. Collective."""
        if self._masks_set or self.world == 1 or self.graph is None:
            return
        need = torch.from_numpy(self.graph.column_use()).to(self.device)
        every = [torch.empty_like(need) for _ in range(self.world)]
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather(every, need, group=self.group)
        else:
            cpu = [torch.empty_like(need, device="cpu") for _ in range(self.world)]
            dist.all_gather(cpu, need.cpu(), group=self.group)
            every = cpu
        mask = np.zeros(self.re - self.rb, np.uint8)
        slot = 0
        for q in range(self.world):
            if q == self.rank:
                continue
            mask |= (every[q][self.rb:self.re].cpu().numpy() != 0).astype(np.uint8) << slot
            slot += 1
        self.graph.set_peer_mask(mask, self.world - 1)
        info = self.graph.info()
        self.exchange_rows, self.exchange_rows_all = int(info.exchange_rows), int(info.exchange_rows_all)
        self._masks_set = True

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

    def map_peer_buffers(self, bufs: list) -> dict:
        """CUDA-IPC map every peer's copies of `bufs` (same shapes on every
        rank). Returns {peer rank: [device pointer of its bufs[i], ...]};
        release with unmap_peer_buffers. Collective."""
        from . import fusedmm as F
        torch.cuda.synchronize(self.device)
        mine = [F.ipc_handle(b.data_ptr()) for b in bufs]
        every: list = [None] * self.world
        dist.all_gather_object(every, mine, group=self.group)
        dev = self.device.index
        self._maps = {}
        # both buffers of a peer may live in one caching-allocator segment
        # (the same handle): map each distinct handle once
        for q in range(self.world):
            if q != self.rank:
                self._maps[q] = {}
                for (h, _off) in every[q]:
                    if h not in self._maps[q]:
                        self._maps[q][h] = F.ipc_open(h, dev)
        return {q: [self._maps[q][h] + off for (h, off) in every[q]] for q in self._maps}

    def unmap_peer_buffers(self) -> None:
        """Collective: no rank unmaps while a peer may still store into it."""
        from . import fusedmm as F
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        for q in getattr(self, "_maps", {}):
            for base in self._maps[q].values():
                F.ipc_close(base)
        self._maps = {}

    def step_exchange(self, X: torch.Tensor, nxt: torch.Tensor, peer_next: list, all_rows: bool = False) -> None:
        """One fused call over this rank's rows of X whose z rows land in
        nxt[rb:re] AND, over NVLink, in every peer's next buffer
        (peer_next[q] = that buffer's device pointer on the peer, rank order
        without self) — only the rows the peer reads unless all_rows — then
        the stream-ordered barrier that makes every slice visible."""
        from ._lib import FMM_ASYNC, FMM_DEVICE_PTRS, FMM_PEERS_ALL, fmm_stats
        row_off = self.rb * self.d * 4
        targets = [p + row_off for p in peer_next]
        st = fmm_stats()
        flags = FMM_DEVICE_PTRS | FMM_ASYNC | (FMM_PEERS_ALL if all_rows else 0)
        self.graph.run_device_peers(X.data_ptr(), X.shape[0], X.data_ptr(), nxt[self.rb:self.re].data_ptr(),
                                    self.d, self.spec, targets, flags=flags, stats=st)
        self.launches += st.launches
        self._barrier()

    def _iterate_fused(self, X0: torch.Tensor, iters: int) -> torch.Tensor:
        if self.halo:
            self.set_halo_masks()
        bufs = [X0.clone(), torch.empty_like(X0)]
        try:
            peers = self.map_peer_buffers(bufs)
            self._barrier()
            for it in range(iters):
                cur, nxt = bufs[it % 2], bufs[(it + 1) % 2]
                # halo rows only, except on the last iteration: the returned
                # iterate is replicated on every rank
                self.step_exchange(cur, nxt, [peers[q][(it + 1) % 2] for q in sorted(peers)],
                                   all_rows=(it + 1 == iters))
            out = bufs[iters % 2]
        finally:
            self.unmap_peer_buffers()
        return out

    def iterate(self, X0: torch.Tensor, iters: int) -> torch.Tensor:
        """iters fused calls with X <- Z; returns the replicated final X."""
        if self.exchange_mode == "fused":
            return self._iterate_fused(X0, iters)
        cur = X0.clone()
        nxt = torch.empty_like(cur)
        for _ in range(iters):
            self._compute(cur, cur, self.rb, self.re, out=nxt[self.rb:self.re])
            self.exchange(nxt)
            cur, nxt = nxt, cur
        return cur
