"""Dev probe: does rendering beside the codec-1 range decode slow the decode?
Times the config-2 codec-1 open (one rc_decode launch, ~527 ms) alone, and
with 300 codec-0 frames rendered on another session's streams at the same
time (the renders' ~57 ms of work would hide under the decode)."""
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
import paper_2509_17513_b200 as g
from paper_2509_17513_b200 import _lib


class A:
    gaussians, layers, frames, group, width, height = 300_000, 6, 300, 30, 1920, 1080


blobs, _ = bench.make_inputs(A, 1002)
cs = _lib.camera_struct(bench.camera(A))
s1, s0 = g.Session(0), g.Session(0)
res = {c: torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda() for c, b in blobs.items()}
info = {c: g.read_structure(b) for c, b in blobs.items()}
outs = [torch.empty((1080, 1920, 3), dtype=torch.float32, device="cuda") for _ in range(300)]
v0 = g.DeviceVideo(blobs[0], 6, session=s0, resident=res[0], info=info[0], group_list=list(range(10)))
v0.render_batch(list(range(300)), cs, outs=outs)
torch.cuda.synchronize()


def open1():
    t0 = time.perf_counter()
    v = g.DeviceVideo(blobs[1], 6, session=s1, resident=res[1], info=info[1], group_list=list(range(10)))
    dt = time.perf_counter() - t0
    v.close()
    return dt * 1e3


for rep in range(2):
    print(f"open codec1 alone: {open1():.1f} ms", flush=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v0.render_batch(list(range(300)), cs, outs=outs, verify=False)  # enqueued, runs beside the decode
    d = open1()
    s0.sync()
    print(f"open codec1 with 300 renders beside: {d:.1f} ms (renders done at {(time.perf_counter() - t0) * 1e3:.1f} ms)",
          flush=True)
    t0 = time.perf_counter()
    v0.render_batch(list(range(300)), cs, outs=outs, verify=False)
    s0.sync()
    print(f"300 renders alone: {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
