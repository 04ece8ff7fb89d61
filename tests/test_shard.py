"""Sharding logic and the multi-process path (world size 2, gloo, CPU)."""

import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_util import container
from oracle import oracle as O
from paper_2509_17513_b200.shard import assign_groups, frames_of, gather_metrics, group_costs


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


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    info = O.read_structure(container("s1_rc"))
    mine = assign_groups(group_costs(info), world)[rank]
    _, groups = O.read_layers(container("s1_rc"), 3)
    # each rank "renders" its own frames (oracle stand-in for the GPU work)
    checks = {}
    for t in frames_of(info, mine):
        g = O.frame_of(groups, t)
        checks[t] = float(g.positions.sum())
    allm = gather_metrics({"rank": rank, "frames": sorted(checks), "sums": checks}, dist)
    if rank == 0:
        q.put(allm)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29517
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    frames = sorted(f for m in res for f in m["frames"])
    assert frames == list(range(6))
    assert {m["rank"] for m in res} == {0, 1}
