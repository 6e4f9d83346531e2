"""Sharding independent scene batches over ranks (BASELINE config C5).

A single scene stays on one GPU. A batch of independent scenes is split into contiguous shards,
one per rank (one process per GPU). Each rank steps its shard as ONE device world
(`SolverHandle.batch`, vrod_batch_create); there is no communication while stepping. The only
collective is the final gather of the per-scene statistics to rank 0 — an all-gather over the
process group (NCCL on GPUs, gloo on CPU).
"""
from __future__ import annotations

import numpy as np

from .workloads import shard_range

STAT_FIELDS = ("r0", "r1", "r2", "r3", "r4", "r5", "r6", "r7", "max_penetration", "contact_count", "broad_pairs",
               "skipped_singular")


def report_rows(reports) -> np.ndarray:
    """Per-scene StepReports -> (n, 12) float64 rows (8 residuals, penetration, 3 counters)."""
    out = np.zeros((len(reports), len(STAT_FIELDS)), dtype=np.float64)
    for i, r in enumerate(reports):
        out[i, :8] = r.residuals
        out[i, 8] = r.max_penetration
        out[i, 9] = r.contact_count
        out[i, 10] = r.broad_pairs
        out[i, 11] = r.skipped_singular
    return out


def gather_scene_stats(rows: np.ndarray, n_total: int, device=None, group=None) -> np.ndarray | None:
    """All-gather every rank's shard rows; rank 0 gets the (n_total, 12) table in scene order.

    Shards are contiguous (`shard_range`), so concatenating rank by rank restores scene order.
    `device`: torch device of the collective (a CUDA device for NCCL, None/CPU for gloo)."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    cap = max(hi - lo for lo, hi in (shard_range(n_total, r, world) for r in range(world)))
    buf = torch.zeros((cap, rows.shape[1]), dtype=torch.float64, device=device)
    buf[: rows.shape[0]] = torch.from_numpy(rows).to(device)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if rank != 0:
        return None
    out = []
    for r, p in enumerate(parts):
        lo, hi = shard_range(n_total, r, world)
        out.append(p[: hi - lo].cpu().numpy())
    return np.concatenate(out, axis=0)
