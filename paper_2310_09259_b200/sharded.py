"""Multi-GPU QUIK linear layer: output-feature (column) sharding + NCCL all-gather.

SURVEY.md §8(e): rank r of g owns weight rows [r*N/g, (r+1)*N/g) with their
scales / wreduced / bias / outlier-weight rows (all indexed by output row only,
runtime.cpp:240, :298-299). x is replicated and K1 runs on every rank; per-token
scale and zero depend only on the full input row, so they need no exchange.
Each rank produces y[:, shard] and one all-gather assembles y [M][N].

K-sharding is rejected (it would need a global per-token min/max all-reduce
before quantisation and an FP32 reduce-scatter of partial outputs).

The collective goes through torch.distributed (backend "nccl" on B200s, "gloo"
in the CPU tests); the per-shard compute is the device QuikLinear.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row range of `rank` (the first n % world ranks get one extra row)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def max_shard(n: int, world: int) -> int:
    return -(-n // world)


def assemble(gathered, n: int, world: int):
    """[world][M][max_shard] (padded shards, rank-major) -> [M][N] row-major.
    Works on numpy arrays and torch tensors."""
    parts = []
    for r in range(world):
        b, e = shard_bounds(n, world, r)
        parts.append(gathered[r][:, : e - b])
    if isinstance(gathered, np.ndarray):
        return np.concatenate(parts, axis=1)
    import torch

    return torch.cat(parts, dim=1)


class ShardedQuikLinear:
    """y = quik_matmul(layer, x) with the output features sharded over a process group.

    layer: the full QuikLinearLayer (host arrays; every rank uploads only its rows).
    compute: optional override of the per-shard compute (tests); defaults to the
    device QuikLinear shard."""

    def __init__(self, layer, group=None, compute: Optional[Callable] = None, device: Optional[int] = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = layer.out_features()
        self.begin, self.end = shard_bounds(self.n, self.world, self.rank)
        self.ns_max = max_shard(self.n, self.world)
        if compute is None:
            from .quik import QuikLinear

            self.local = QuikLinear(layer, device=device, row_begin=self.begin, row_end=self.end)
            self.compute = lambda x: self.local(x)
        else:
            self.compute = compute

    def forward(self, x):
        import torch

        y_local = self.compute(x)  # [M][end - begin]
        M = y_local.shape[0]
        pad = torch.zeros((M, self.ns_max), dtype=y_local.dtype, device=y_local.device)
        pad[:, : self.end - self.begin] = y_local
        gathered = torch.empty((self.world * M, self.ns_max), dtype=y_local.dtype, device=y_local.device)
        self.dist.all_gather_into_tensor(gathered, pad, group=self.group)
        return assemble(gathered.view(self.world, M, self.ns_max), self.n, self.world)

    __call__ = forward


# --------------------------------------------------------------------------- fused all-gather (CUDA IPC)


def gather_handles(mine: list, group=None) -> list:
    """Every rank's list of serialised IPC handles (one per output buffer), rank-indexed."""
    import torch.distributed as dist

    allh = [None] * dist.get_world_size(group)
    dist.all_gather_object(allh, mine, group=group)
    return allh


def peer_destinations(rank: int, world: int, own, opened: dict) -> list:
    """Destination list of a rank's fused epilogue: its own output first, then every
    other rank's output (opened IPC mappings) in rank order."""
    if set(opened) != set(range(world)) - {rank}:
        raise ValueError("fused all-gather: need the outputs of every other rank")
    return [own] + [opened[r] for r in range(world) if r != rank]


class FusedAllGatherOutput:
    """[M][N] f16 output buffers shared by all ranks of a process group through CUDA IPC
    (one process per GPU): every rank's GEMM epilogue TMA-stores its
    shard tile by tile into EVERY rank's buffer (C ABI quik_linear_forward_sharded), so
    the exchange rides NVLink under the next tiles' MMAs and needs no all-gather or
    transpose. `buffers` outputs are used round robin: with two, the completion
    barrier of step i also orders every rank's readers of step i-2's buffer (enqueued
    before step i-1) before step i's writes into it."""

    def __init__(self, M: int, N: int, group=None, device=None, buffers: int = 2, barrier_fn=None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _lib
        from .quik import context

        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.lib = _lib.load()
        self.ctx = context(device)
        dev = torch.device("cuda", self.ctx.device)
        self.bufs = [torch.empty((M, N), dtype=torch.float16, device=dev) for _ in range(buffers)]
        mine = []
        for b in self.bufs:
            h = _lib.IpcHandle()
            _lib.check(self.lib.quik_ipc_handle_get(self.ctx.handle, C.c_void_p(b.data_ptr()), C.byref(h)))
            mine.append(bytes(h.bytes) + int(h.offset).to_bytes(8, "little", signed=True))
        allh = gather_handles(mine, group)
        self._opened = []  # (ptr, handle) to close
        self.dests = []
        for i, b in enumerate(self.bufs):
            opened = {}
            for r in range(self.world):
                if r == self.rank:
                    continue
                raw = allh[r][i]
                h = _lib.IpcHandle()
                C.memmove(h.bytes, raw[:64], 64)
                h.offset = int.from_bytes(raw[64:72], "little", signed=True)
                p = C.c_void_p()
                _lib.check(self.lib.quik_ipc_handle_open(self.ctx.handle, C.byref(h), C.byref(p)))
                opened[r] = p.value
                self._opened.append((p.value, h))
            self.dests.append(peer_destinations(self.rank, self.world, b.data_ptr(), opened))
        self.flag = torch.zeros(1, dtype=torch.float32, device=dev)
        self.step = 0
        self._barrier_fn = barrier_fn

    def next(self):
        """-> (buffer index, destination pointers) of the next step."""
        i = self.step % len(self.bufs)
        self.step += 1
        return i, self.dests[i]

    def barrier(self):
        """Stream-ordered completion fence: every rank's stores into every buffer are done
        (a one-element all-reduce on the group, after the GEMM in stream order)."""
        if self._barrier_fn is not None:
            self._barrier_fn()
            return
        self.dist.all_reduce(self.flag, group=self.group)

    def close(self):
        import ctypes as C

        for p, h in self._opened:
            self.lib.quik_ipc_handle_close(self.ctx.handle, C.c_void_p(p), C.byref(h))
        self._opened = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class FusedShardedQuikLinear:
    """y = quik_matmul(layer, x) over a process group with the all-gather fused into the
    GEMM epilogue (CUDA IPC peer stores, FusedAllGatherOutput). Returns this rank's copy
    of the full [M][N] f16 output (valid on the current stream after the barrier)."""

    def __init__(self, layer, max_tokens: int, group=None, device=None, local=None, n_total: int = 0,
                 barrier: bool = True, barrier_fn=None):
        """layer: the full QuikLinearLayer (host arrays), or local = this rank's device
        shard (QuikLinear over rows shard_bounds(n_total, world, rank)) + n_total."""
        import torch.distributed as dist

        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        self.n = layer.out_features() if local is None else n_total
        self.begin, self.end = shard_bounds(self.n, world, rank)
        if local is None:
            from .quik import QuikLinear

            local = QuikLinear(layer, device=device, row_begin=self.begin, row_end=self.end)
        self.local = local
        self.out = FusedAllGatherOutput(max_tokens, self.n, group=group, device=local.device, barrier_fn=barrier_fn)
        self.use_barrier = barrier

    def forward(self, x):
        i, dests = self.out.next()
        buf = self.out.bufs[i]
        M = x.shape[0]
        self.local.forward_sharded_ptrs(x, dests, buf.stride(0), self.begin)
        if self.use_barrier:
            self.out.barrier()
        return buf[:M]

    __call__ = forward
