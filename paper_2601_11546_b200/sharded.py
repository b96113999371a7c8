"""Sharded pool across processes (BASELINE config 5).

One process per GPU.  Every rank builds the same trace, creates its shard
(`Engine(..., shards=world, shard_rank=rank)`), and the ranks swap the CUDA IPC
handles of their mailboxes over the process group (any torch.distributed
backend: this is bootstrap plumbing, not the per-iteration exchange, which the
persistent kernel does itself over NVLink peer memory; csrc/shard.cuh).
"""

from __future__ import annotations


def exchange_handles(local_handle: bytes, group=None) -> list[bytes]:
    """All-gather every rank's 64-byte mailbox handle, in rank order."""
    import torch.distributed as dist

    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, local_handle, group=group)
    for r, h in enumerate(out):
        if not isinstance(h, (bytes, bytearray)) or len(h) != 64:
            raise RuntimeError(f"rank {r} sent a malformed mailbox handle")
    return [bytes(h) for h in out]


def connect(engine, group=None) -> None:
    """Connect this rank's shard engine to every other rank's (collective)."""
    engine.connect_shards(exchange_handles(engine.mailbox_handle(), group))


def run_sharded(trace, policy, world_model, config=None, policy_model=None, seed: int = 0, *, group=None,
                device: int | None = None):
    """`run(...)` (engine.py:466-475) with the relQueries sharded over the process group's ranks."""
    import torch.distributed as dist

    from .engine import Engine

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if device is None:
        import torch

        device = torch.cuda.current_device()
    eng = Engine(trace, policy, world_model, config, policy_model, seed, device=device, shards=world,
                 shard_rank=rank)
    try:
        connect(eng, group)
        return eng.run()
    finally:
        eng.close()
