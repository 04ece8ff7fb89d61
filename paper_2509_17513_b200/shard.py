"""Multi-GPU sharding of a container's frames (one process per GPU).

A motion group (container.py:54-70) is the unit of work: codec-1 runs are
sequential inside a group (codec.py:183-223), so a group is decoded by one
rank; codec-0 frames and camera views need no exchange at all.  Groups are
assigned by longest-processing-time first on frames x splats, which
balances the adaptive (variable-length) groups of BASELINE config 3.  No
collective is needed on the data path; `gather_metrics` all-gathers the
per-rank results afterwards (NCCL over NVLink on the GPU box, gloo in the CPU
tests).
"""

from __future__ import annotations

import heapq
from typing import Sequence


def group_costs(info, up_to_layer: int | None = None) -> list:
    """frames x splats of every group at the layer prefix."""
    k = info.layer_count if up_to_layer is None else up_to_layer
    return [int(g.frame_count) * int(sum(g.layer_counts[:k])) for g in info.groups]


def assign_groups(costs: Sequence[int], world: int) -> list:
    """LPT assignment: list (per rank) of group indices, each sorted."""
    if world < 1:
        raise ValueError("world must be >= 1")
    heap = [(0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for g in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        load, r = heapq.heappop(heap)
        out[r].append(g)
        heapq.heappush(heap, (load + costs[g], r))
    return [sorted(x) for x in out]


def frames_of(info, groups: Sequence[int]) -> list:
    """Global frame indices of the given groups, ascending."""
    fr = []
    for g in groups:
        gd = info.groups[g]
        fr.extend(range(gd.start_frame, gd.start_frame + gd.frame_count))
    return sorted(fr)


def gather_metrics(values: dict, dist) -> list:
    """All-gather a small per-rank metrics dict (after the timed region)."""
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, values)
    return out
