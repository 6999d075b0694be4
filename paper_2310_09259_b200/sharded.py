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
