"""Scene-parallel batches across GPUs (BASELINE config 5).

A single garment is never sharded.  Independent scenes are partitioned
statically, one process per GPU, with no collective on the hot path: each
rank steps its own scenes and only per-scene metrics are gathered at the end
(``gather_metrics``, any torch.distributed backend - NCCL on the GPU box,
gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np


def scene_shard(n_scenes: int, world: int, rank: int) -> range:
    """Contiguous block of scene ids owned by `rank` (balanced to +-1)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(n_scenes, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def gather_metrics(local: dict, world: int, device: str = "cpu") -> dict:
    """All-gather per-scene metric rows {scene_id: [values...]} to every rank."""
    if world == 1:
        return dict(local)
    import torch
    import torch.distributed as dist

    ids = sorted(local)
    width = len(next(iter(local.values()))) if local else 0
    counts = torch.tensor([len(ids)], device=device)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts)
    cap = int(max(int(c) for c in all_counts))
    buf = torch.full((cap, width + 1), float("nan"), dtype=torch.float64, device=device)
    for r, sid in enumerate(ids):
        buf[r, 0] = sid
        buf[r, 1:] = torch.as_tensor(np.asarray(local[sid], dtype=np.float64))
    out = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    merged = {}
    for t in out:
        for row in t.cpu().numpy():
            if not np.isnan(row[0]):
                merged[int(row[0])] = row[1:].tolist()
    return merged
