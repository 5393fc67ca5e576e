"""Multi-GPU partitioning of the hot path.

Domains ((layer, KV head) pairs, the reference's layer_id space) are independent: each rank owns a
contiguous block of domains with its own ClusterKVCache (its own index / store / maintainer), so
ingest needs no exchange; a decode step ends with one all-gather of the per-domain outputs
(D x d values) in rank order. Streams (config 5) are independent too: rank r serves streams
r, r + world, ... with no collective at all.
"""
from __future__ import annotations


def shard_domains(n_domains: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) of the domains rank `rank` owns (contiguous, balanced, rank-ordered)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world / rank")
    if n_domains < world:
        raise ValueError(f"{n_domains} domains cannot be split over {world} ranks")
    base, extra = divmod(n_domains, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_streams(n_streams: int, world: int, rank: int) -> list[int]:
    """Streams served by `rank` (round robin; independent, no collective)."""
    return list(range(rank, n_streams, world))


def gather_domain_outputs(out_local, n_domains: int, group=None):
    """All-gather per-domain outputs [D_local, d] into [n_domains, d] in domain order.

    Uses torch.distributed (NCCL over NVLink on GPUs, gloo in CPU tests). Ranks may own unequal
    blocks; they are padded to the largest block for the collective and trimmed afterwards.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    d = out_local.shape[-1]
    blocks = [shard_domains(n_domains, world, r) for r in range(world)]
    width = max(b - a for a, b in blocks)
    pad = torch.zeros(width, d, dtype=out_local.dtype, device=out_local.device)
    pad[: out_local.shape[0]] = out_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[: b - a] for p, (a, b) in zip(parts, blocks)], dim=0)


class FusedExchange:
    """Fused output exchange (kvc_set_peers): the attention kernel writes every finished output row
    into every rank's exchange buffer over peer memory (NVLink P2P stores through CUDA IPC
    mappings), replacing the per-step all-gather; only the 64-byte IPC handles go through the
    process group (once). After kv.query, `gathered(out)` yields all domains' outputs."""

    def __init__(self, kv, n_domains: int, group=None):
        import torch.distributed as dist

        from .api import ipc_alloc, ipc_open, lib

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.kv = kv
        self.n_domains = n_domains
        a, b = shard_domains(n_domains, self.world, self.rank)
        if b - a != kv.L:
            raise ValueError("the context must hold exactly this rank's domain block")
        nbytes = int(lib().kvc_exchange_bytes(self.world, n_domains, kv.d))
        self.own, handle = ipc_alloc(nbytes)
        handles = [None] * self.world
        dist.all_gather_object(handles, handle, group=group)
        self.bufs = [self.own if r == self.rank else ipc_open(handles[r]) for r in range(self.world)]
        dist.barrier(group=group)
        kv.set_peers(self.world, self.rank, a, n_domains, self.bufs)

    def gathered(self, out):
        return self.kv.peer_output(out)
