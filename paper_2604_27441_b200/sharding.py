"""Multi-GPU layout: independent conference streams shard across GPUs.

SURVEY.md 8(e): stream s is owned by GPU ``s mod G``; each owner keeps the
stream's k-frame reference ring resident and batches its streams of equal
shape into one ``nvrec_recover_u8`` launch per modality.  There is no
collective on the data path -- ``torch.distributed`` is used only for the
benchmark's barrier and max-over-ranks timing.
"""

from __future__ import annotations


def owner(stream_id: int, world: int) -> int:
    """Rank (GPU) that serves ``stream_id``."""
    return stream_id % world


def streams_for_rank(n_streams: int, rank: int, world: int) -> list[int]:
    """Stream ids served by ``rank`` (ascending)."""
    return [s for s in range(n_streams) if owner(s, world) == rank]


def route(requests, world: int) -> dict[int, list]:
    """Group ``(stream_id, payload)`` requests by owning rank, preserving
    per-stream order (frames of one stream must be recovered in order since
    each recovered plane joins that stream's reference ring)."""
    out: dict[int, list] = {r: [] for r in range(world)}
    for sid, payload in requests:
        out[owner(sid, world)].append((sid, payload))
    return out
