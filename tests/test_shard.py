"""Sharding of one sequence over ranks (shard.py) and the multi-process path.

CPU: the plans (contiguous equal-cost frame ranges for raw groups, LPT over
whole groups for range-coded ones), the raw/sequential classification of the
reference's own containers, and a world-size-2 gloo run in which every rank
computes its plan and the all-gathered union covers every frame exactly once.

GPU: the product path with two ranks sharing the one GPU under gloo -- each
rank opens only its groups (gsv_video_open_group_list) and renders only its
frames; the all-gathered frames equal a single-process render of the whole
sequence bit for bit.
"""

import os
from types import SimpleNamespace as NS

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_util import container
from oracle import oracle as O
from paper_2509_17513_b200.shard import (assign_groups, frames_of, gather_metrics, global_frames,
                                         group_costs, local_frames, pieces_groups, plan, raw_groups)


def test_lpt_balances_and_covers():
    costs = [30, 2, 2, 2, 10, 10, 9, 1]
    parts = assign_groups(costs, 3)
    assert sorted(g for p in parts for g in p) == list(range(len(costs)))
    loads = [sum(costs[g] for g in p) for p in parts]
    assert max(loads) == 30 and min(loads) >= 14
    assert assign_groups([5], 4)[0] == [0] and assign_groups([5], 4)[1:] == [[], [], []]


def test_frames_of_reference_container():
    info = O.read_structure(container("deg0_rc"))
    parts = assign_groups(group_costs(info), 2)
    frames = sorted(f for p in parts for f in frames_of(info, p))
    assert frames == list(range(sum(g.frame_count for g in info.groups)))


def _c2_info(groups=10, frames=30, n=50_000):
    return NS(layer_count=6, groups=[NS(frame_count=frames, start_frame=frames * i, layer_counts=[n] * 6)
                                     for i in range(groups)])


@pytest.mark.parametrize("world", [1, 2, 3, 4, 7, 8])
def test_plan_raw_sequence_contiguous_equal(world):
    """Codec 0 (every group raw): N contiguous frame ranges, sizes within one
    frame of each other, covering the sequence once, in order."""
    info = _c2_info()
    parts = plan(info, world, [True] * 10)
    sizes = [len(global_frames(info, p)) for p in parts]
    assert max(sizes) - min(sizes) <= 1 and sum(sizes) == 300
    allf = [f for p in parts for f in global_frames(info, p)]
    assert allf == list(range(300))
    for p in parts:  # local numbering inside the opened group list
        loc, gl = local_frames(info, p), pieces_groups(p)
        starts = np.cumsum([0] + [info.groups[g].frame_count for g in gl])
        for lf, gf in zip(loc, global_frames(info, p)):
            gi = int(np.searchsorted(starts, lf, side="right") - 1)
            assert info.groups[gl[gi]].start_frame + (lf - starts[gi]) == gf


def test_plan_sequential_groups_whole():
    """Range-coded groups stay whole (LPT): 10 equal groups on 8 ranks."""
    info = _c2_info()
    parts = plan(info, 8, [False] * 10)
    assert all(p.f0 == 0 and p.f1 == 30 for ps in parts for p in ps)
    assert sorted(p.group for ps in parts for p in ps) == list(range(10))
    assert sorted(len(ps) for ps in parts) == [1] * 6 + [2] * 2


def test_plan_uneven_layer_sizes_weighted():
    """Frames of groups with more splats weigh more."""
    info = NS(layer_count=1, groups=[NS(frame_count=10, start_frame=0, layer_counts=[300]),
                                     NS(frame_count=10, start_frame=10, layer_counts=[100])])
    parts = plan(info, 2, [True, True])
    cost = [sum(info.groups[p.group].layer_counts[0] * (p.f1 - p.f0) for p in ps) for ps in parts]
    assert abs(cost[0] - cost[1]) <= 300


def test_raw_groups_classification():
    raw = container("s1_raw")
    rc = container("s1_rc")
    assert all(raw_groups(raw, O.read_structure(raw)))
    assert not all(raw_groups(rc, O.read_structure(rc)))


def _plan_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    for name in ("s1_raw", "s1_rc"):
        data = container(name)
        info = O.read_structure(data)
        mine = plan(info, world, raw_groups(data, info))[rank]
        out[name] = global_frames(info, mine)
    allm = gather_metrics({"rank": rank, "frames": out}, dist)
    if rank == 0:
        q.put(allm)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_plans_cover_sequence():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_plan_worker, args=(r, 2, 29517, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for name in ("s1_raw", "s1_rc"):
        info = O.read_structure(container(name))
        total = sum(g.frame_count for g in info.groups)
        frames = sorted(f for m in res for f in m["frames"][name])
        assert frames == list(range(total)), name
        assert all(m["frames"][name] for m in res)  # both ranks got work
    assert {m["rank"] for m in res} == {0, 1}


# ---------------------------------------------------------------------------
def _gpu_worker(rank, world, port, q, name, k):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import torch

    import paper_2509_17513_b200 as g
    from golden_util import camera
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    data = container(name)
    info = g.read_structure(data)
    mine = plan(info, world, raw_groups(data, info, k), k)[rank]
    cam = camera(name, "oblique")
    imgs = {}
    with g.DeviceVideo(data, k, group_list=pieces_groups(mine)) as v:
        for lf, gf in zip(local_frames(info, mine), global_frames(info, mine)):
            imgs[gf] = v.render(lf, cam).cpu().numpy()
    got = [None] * world
    dist.all_gather_object(got, {"rank": rank, "imgs": imgs})
    if rank == 0:
        q.put(got)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["s1_raw", "s1_rc"])
def test_two_ranks_one_gpu_product_path(name):
    """Two ranks (gloo, sharing cuda:0) each decode and render only their
    shard of a reference container through the C ABI; the union of their
    frames equals a single-process render of every frame, bit for bit."""
    import paper_2509_17513_b200 as g
    from golden_util import camera
    k = O.read_structure(container(name)).layer_count
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, 29531 + len(name), q, name, k)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    union = {}
    for m in res:
        assert m["imgs"], "every rank renders part of the sequence"
        for t, img in m["imgs"].items():
            assert t not in union
            union[t] = img
    cam = camera(name, "oblique")
    with g.DeviceVideo(container(name), k) as v:
        assert sorted(union) == list(range(v.frame_count))
        for t in range(v.frame_count):
            assert np.array_equal(union[t], v.render(t, cam).cpu().numpy()), t


def _bench_dist_worker(rank, world, port, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import torch

    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RANK"], os.environ["WORLD_SIZE"] = str(rank), str(world)
    d = bench.Dist(world, rank, use_cuda=False)  # no GPU here: gloo, host tensors
    d.barrier()
    mx = d.max(float(rank + 1) * 1.5)
    objs = d.objects({"rank": rank, "frames": list(range(rank, 10, world))})
    frames = d.tensors(torch.full((4, 6, 3), rank, dtype=torch.uint8))
    if rank == 0:
        q.put({"backend": d.backend, "max": mx, "objs": objs, "frames": [f.tolist() for f in frames]})
    d.barrier()
    d.close()


def test_bench_dist_gloo_two_ranks():
    """bench.py's torch.distributed plumbing (the max-over-ranks timing, the
    per-rank metric gather and the sampled-frame gather) at world size 2."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_bench_dist_worker, args=(r, 2, 29533, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res["backend"] == "gloo" and res["max"] == 3.0
    assert [o["rank"] for o in res["objs"]] == [0, 1]
    assert sorted(f for o in res["objs"] for f in o["frames"]) == list(range(10))
    assert [np.unique(np.array(f)).tolist() for f in res["frames"]] == [[0], [1]]
