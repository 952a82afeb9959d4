"""Keyframe sharding for the multi-GPU step.

The batch mean of total_objective (objective.cpp:77: inv_b = 1 / batch size) must use the
GLOBAL batch size on every rank; each rank renders / decodes / back-propagates its own
frames, the gradient buffer and the per-frame loss partials are summed with one all-reduce,
and the trust-region term (objective.cpp:247-256) enters once (rank 0)."""
from __future__ import annotations


def shard_frames(nframes: int, world: int, rank: int):
    """Contiguous split of the keyframe window; returns (first_global_index, count)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(nframes, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


def rank_plan(nframes: int, world: int, rank: int):
    """What a rank hands to latmap_session_set_batch / set_slot_offset."""
    first, count = shard_frames(nframes, world, rank)
    return {"frames": list(range(first, first + count)), "global_batch": nframes,
            "add_trust": rank == 0, "slot_offset": first}
