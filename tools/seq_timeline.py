"""Dev: one render_sequence call on the config-2 codec-0 container with
GSV_DEBUG_SEQ_TIMING=1 (per-group timeline of the pipeline on stderr)."""
import os
import sys
import time
from pathlib import Path

os.environ["GSV_DEBUG_SEQ_TIMING"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
import paper_2509_17513_b200 as g
from paper_2509_17513_b200 import _lib


class A:
    gaussians, layers, frames, group, width, height = 300_000, 6, 300, 30, 1920, 1080


blobs, _ = bench.make_inputs(A, 1002)
data = blobs[0]
info = g.read_structure(data)
cs = _lib.camera_struct(bench.camera(A))
sess = g.Session(0)
hsrc = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
pinned = torch.empty((300, 1080, 1920, 3), dtype=torch.uint8).pin_memory()
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    t0 = time.perf_counter()
    g.render_sequence(hsrc, cs, up_to_layer=6, out=pinned, session=sess, info=info)
    print(f"call {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms", file=sys.stderr, flush=True)
