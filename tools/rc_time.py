"""Codec-1 decode timing at full config-2 scale (dev tool): open the
300-frame container (10 groups, 1380 runs, resident in HBM) with each range
decoder variant, CUDA-event time of the open (decode + CRC), and check the
variants' decoded codes agree on a few frames.

usage: rc_time.py [variants...]   (default 3 4)"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
import paper_2509_17513_b200 as g


class A:
    gaussians, layers, frames, group, width, height = 300_000, 6, 300, 30, 1920, 1080


variants = sys.argv[1:] or ["3", "4"]
blobs, _ = bench.make_inputs(A, 1002)
data = blobs[1]
res = torch.empty(len(data) + 64, dtype=torch.uint8, device="cuda")
res[:len(data)].copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
info = g.read_structure(data)
sess = g.Session()
codes = {}
for v in variants:
    os.environ["GSV_RC_VARIANT"] = v
    times = []
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sess.stream)
        vid = g.DeviceVideo(data, 6, session=sess, resident=res, info=info)
        e1.record(sess.stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        if rep == 0:
            codes[v] = [vid.frame_codes(t).cpu() for t in (1, 29, 150, 299)]
        vid.close()
    print(f"variant {v}: open (decode + CRC) {min(times):.1f} ms (runs of {times})", flush=True)
ref = codes[variants[0]]
for v in variants[1:]:
    same = all(torch.equal(a, b) for a, b in zip(ref, codes[v]))
    print(f"variant {v} codes == variant {variants[0]}: {same}")
