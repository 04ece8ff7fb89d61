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


# ---------------------------------------------------------------------------
# Shard plans: which frames of which groups a rank decodes and renders.
class Piece(tuple):
    """(group, f0, f1): frames [f0, f1) of container group `group` (group-relative)."""

    __slots__ = ()

    def __new__(cls, group: int, f0: int, f1: int):
        return super().__new__(cls, (int(group), int(f0), int(f1)))

    group = property(lambda self: self[0])
    f0 = property(lambda self: self[1])
    f1 = property(lambda self: self[2])


def raw_groups(data, info, up_to_layer: int | None = None) -> list:
    """Per group: True when every run of layers <= k is stored raw (codec 0,
    or codec 1's whole-run raw fallback, codec.py:137-163): its planes stand
    alone, so the group's frames can be split between ranks.  A group with a
    range-coded run decodes sequentially (codec.py:183-223) and stays whole."""
    k = info.layer_count if up_to_layer is None else up_to_layer
    out = []
    for g in info.groups:
        raw = True
        for l in range(k):
            for e in g.channels[l]:
                head = bytes(data[e.offset:e.offset + 15])
                if len(head) < 15 or not (head[0] == 0 or (head[0] == 1 and head[14] == 1)):
                    raw = False
        out.append(raw)
    return out


def plan(info, world: int, splittable=None, up_to_layer: int | None = None) -> list:
    """Assign a sequence's frames to `world` ranks; returns per rank a list of
    Pieces in sequence order.

    splittable[g] (default: all False) says whether group g's frames may be
    split (raw runs).  When every group is splittable the sequence is cut into
    `world` contiguous frame ranges of equal cost (splats per frame), the
    exact balance codec 0 allows; otherwise groups stay whole and are
    assigned by longest-processing-time on frames x splats (assign_groups)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    k = info.layer_count if up_to_layer is None else up_to_layer
    G = len(info.groups)
    split = list(splittable) if splittable is not None else [False] * G
    if G and all(split):
        per = [int(sum(g.layer_counts[:k])) for g in info.groups]
        total = sum(per[g] * info.groups[g].frame_count for g in range(G))
        out = [[] for _ in range(world)]
        acc = 0
        for g, gd in enumerate(info.groups):
            for f in range(gd.frame_count):
                # the rank owning this frame's cost midpoint
                r = min(world - 1, int((2 * acc + per[g]) * world // (2 * total))) if total else 0
                acc += per[g]
                lst = out[r]
                if lst and lst[-1].group == g and lst[-1].f1 == f:
                    lst[-1] = Piece(g, lst[-1].f0, f + 1)
                else:
                    lst.append(Piece(g, f, f + 1))
        return out
    parts = assign_groups(group_costs(info, k), world)
    return [[Piece(g, 0, info.groups[g].frame_count) for g in p] for p in parts]


def pieces_groups(pieces) -> list:
    """Distinct groups of a rank's pieces, in order (the group list it opens)."""
    seen, out = set(), []
    for p in pieces:
        if p.group not in seen:
            seen.add(p.group)
            out.append(p.group)
    return out


def local_frames(info, pieces) -> list:
    """Frame numbers inside a video opened with pieces_groups(pieces)
    (frames numbered group after group in list order) of every piece frame."""
    base, acc = {}, 0
    for g in pieces_groups(pieces):
        base[g] = acc
        acc += info.groups[g].frame_count
    return [base[p.group] + f for p in pieces for f in range(p.f0, p.f1)]


def global_frames(info, pieces) -> list:
    """Sequence frame numbers (DecodedVideo.frame(t) numbering) of the pieces."""
    return [info.groups[p.group].start_frame + f for p in pieces for f in range(p.f0, p.f1)]
