"""Dev diagnostic: where a bench step's time goes (config 2, codec 0, k = 6,
container resident).  Times, per step (5 steps after 2 warm-up):
  full   open + render_batch(300 frames) + close   (the bench step)
  open   open + close only (stage tables, CRC of every run, sync)
  render render_batch(300 frames) on a video opened once
and the host-side share of each (wall time of the call without waiting)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
import paper_2509_17513_b200 as g
from paper_2509_17513_b200 import _lib


class A:
    gaussians, layers, frames, group, width, height = 300_000, 6, 300, 30, 1920, 1080


codec = int(sys.argv[1]) if len(sys.argv) > 1 else 0
blobs, _ = bench.make_inputs(A, 1002)
data = blobs[codec]
res = torch.empty(len(data) + 64, dtype=torch.uint8, device="cuda")
res[:len(data)].copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
info = g.read_structure(data)
cs = _lib.camera_struct(bench.camera(A))
sess = g.Session(0)
outs = [torch.empty((1080, 1920, 3), dtype=torch.float32, device="cuda") for _ in range(300)]
groups = list(range(len(info.groups)))


def full():
    v = g.DeviceVideo(data, 6, session=sess, resident=res, info=info, group_list=groups)
    v.render_batch(list(range(300)), cs, outs=outs, verify=False)
    v.close()


def open_only():
    v = g.DeviceVideo(data, 6, session=sess, resident=res, info=info, group_list=groups)
    v.close()


vopen = g.DeviceVideo(data, 6, session=sess, resident=res, info=info, group_list=groups)


def render_only():
    vopen.render_batch(list(range(300)), cs, outs=outs, verify=False)


def render30():
    vopen.render_batch(list(range(30)), cs, outs=outs[:30], verify=False)


hsrc = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
pinned = torch.empty((300, 1080, 1920, 3), dtype=torch.uint8).pin_memory()


def seq_e2e():
    g.render_sequence(hsrc, cs, up_to_layer=6, out=pinned, session=sess, info=info)


def seq_res():
    g.render_sequence(data, cs, up_to_layer=6, resident=res, outs=outs, session=sess, info=info)


for name, fn in (("full", full), ("open", open_only), ("render", render_only), ("render30", render30),
                 ("seq_e2e", seq_e2e), ("seq_res", seq_res), ("full", full), ("seq_res", seq_res)):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    host = 0.0
    for _ in range(5):
        t1 = time.perf_counter()
        fn()
        host += time.perf_counter() - t1
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 5 * 1e3
    print(f"{name:7s} {wall:8.2f} ms/step  host-in-call {host / 5 * 1e3:8.2f} ms", flush=True)
