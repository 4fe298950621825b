"""Sequence sharding of one decode layer across the GPUs of a node.

Membership q·k >= tau is independent per key, so a contiguous partition of the
context gives per-shard selected sets whose union is the global set (no
cross-shard bounds). Each rank probes, filters and attends its own shard and
emits per-q-head partials (m, l, o[d]) with o unnormalised; one all-gather of
[world][rows][d+2] fp32 partials and a log-sum-exp combine (lv_lse_merge, an
sm_100a kernel) give the exact attention over the whole context. New keys of a
decode step go to the last shard, which owns the tail and the update buffer, so
buffer semantics (cache.cpp:7-70) are those of a single cache.
"""
from typing import Optional, Tuple


def shard_range(n_total: int, world: int, rank: int) -> Tuple[int, int]:
    """(first, count) of rank's contiguous slice of [0, n_total); sizes differ by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: 0 <= rank < world required")
    if n_total < 0:
        raise ValueError("shard_range: n_total >= 0 required")
    base, extra = divmod(n_total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def insert_owner(world: int) -> int:
    """Rank that appends decode-step keys (the tail shard, holder of the buffer)."""
    return world - 1


def gather_partials(part, group=None):
    """All-gather one rank's partials [rows][d+2] into [world][rows][d+2] (rank order).
    NCCL gathers device tensors in place; with a CPU backend (gloo) device partials are
    staged through host memory and the result is returned on the partials' device."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    staged = part.is_cuda and dist.get_backend(group) != "nccl"
    src = part.cpu() if staged else part
    out = src.new_empty((world,) + tuple(src.shape))
    try:
        dist.all_gather_into_tensor(out, src.contiguous(), group=group)
    except (RuntimeError, NotImplementedError, ValueError):  # backends without the fused collective
        dist.all_gather(list(out.unbind(0)), src.contiguous(), group=group)
    return out.to(part.device, non_blocking=False) if staged else out


class ShardedLayer:
    """One rank's shard of a decode layer: query -> partial -> all-gather -> LSE merge.

    ``layer`` is this rank's LouverLayer over keys shard_range(n_total, world, rank).
    """

    def __init__(self, layer, group=None):
        import torch.distributed as dist

        self.layer = layer
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def push_key(self, k, v, stream=None) -> None:
        """One decode step's key/value per slot: appended by the tail shard only (it owns the
        update buffer, so flush-at-B behaves as in one cache, cache.cpp:7-10)."""
        if self.rank == insert_owner(self.world):
            self.layer.push_key(k, v, stream=stream)

    def query(self, q, tau, out, *, strict: bool = False, partial: Optional[object] = None, sel_bits=None):
        import torch

        from .louver import lse_merge

        rows = out.shape[0] * out.shape[1]
        d = out.shape[2]
        if partial is None:
            partial = torch.empty((out.shape[0], out.shape[1], d + 2), dtype=torch.float32, device=out.device)
        self.layer.query_device(q, tau, None, strict=strict, partial=partial, sel_bits=sel_bits)
        gathered = gather_partials(partial.view(rows, d + 2), self.group)
        lse_merge(gathered, out.view(rows, d))
        return out
