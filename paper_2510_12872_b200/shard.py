"""Layer sharding of the realignment across the GPUs of one box.

Every (layer, KV-head, token) unit of a4/a5 is independent and the matching
weights depend only on (sample, pool), so each rank holds a contiguous block of
layers of every pool and base cache, computes the weights redundantly from the
replicated embeddings, and realigns its block with no communication.  The only
exchange is the targeted gather of each consuming agent's realigned cache onto the
GPU that prefills/decodes that agent: agent m lives on rank (m-1) mod G and
receives the G layer blocks of its prompt cache (NCCL grouped send/recv through
torch.distributed; no all-gather, which would move G times the bytes).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import torch
import torch.distributed as dist


def layer_shard(num_layers: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [begin, end) layer block of `rank`; sizes differ by at most one."""
    if not (0 <= rank < world) or world < 1:
        raise ValueError("bad rank/world")
    base, rem = divmod(num_layers, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def consumer_rank(agent: int, world: int) -> int:
    """GPU that hosts agent m (1-based): (m - 1) mod G."""
    return (agent - 1) % world


def gather_to_consumers(agents: Sequence[int], shards: Sequence[Tuple[torch.Tensor, torch.Tensor]],
                        full: Sequence[Tuple[torch.Tensor, torch.Tensor]], num_layers: int, rank: int,
                        world: int, group=None) -> None:
    """Targeted gather: for each agent, every rank's layer block of (K, V) lands in
    the consumer rank's full [L, Hs, N, d] buffers.

    shards[i] = (K, V) of agents[i] on this rank, [Ls, Hs, N, d]
    full[i]   = (K, V) full-depth buffers on the consumer rank (ignored elsewhere)
    """
    staged = dist.get_backend(group) == "gloo" and any(
        t is not None and t.is_cuda for pair in shards for t in pair)
    if staged:   # gloo moves host tensors only: stage through host memory (test path)
        cpu_full = [(f[0].cpu(), f[1].cpu()) if f[0] is not None else (None, None) for f in full]
        gather_to_consumers(agents, [(k.cpu(), v.cpu()) for k, v in shards], cpu_full, num_layers, rank, world,
                            group)
        for f, c in zip(full, cpu_full):
            if f[0] is not None:
                f[0].copy_(c[0])
                f[1].copy_(c[1])
        return
    ops = []
    for i, m in enumerate(agents):
        dst = consumer_rank(m, world)
        kb, vb = shards[i]
        if rank == dst:
            for src in range(world):
                lb, le = layer_shard(num_layers, src, world)
                if src == rank:
                    full[i][0][lb:le].copy_(kb)
                    full[i][1][lb:le].copy_(vb)
                else:
                    ops.append(dist.P2POp(dist.irecv, full[i][0][lb:le], src, group))
                    ops.append(dist.P2POp(dist.irecv, full[i][1][lb:le], src, group))
        else:
            ops.append(dist.P2POp(dist.isend, kb, dst, group))
            ops.append(dist.P2POp(dist.isend, vb, dst, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
