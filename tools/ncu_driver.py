"""Small driver for ncu captures: one 30-frame group of the config-2 scene,
decode (codec 0 and 1) and render a few 1080p frames (dev tool)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
import paper_2509_17513_b200 as g
from paper_2509_17513_b200 import _lib

class A:
    gaussians, layers, frames, group, width, height = 300_000, 6, 30, 30, 1920, 1080

codecs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "01")]
blobs, _ = bench.make_inputs(A, 1002)
cam = bench.camera(A)
cs = _lib.camera_struct(cam)
for c in codecs:
    v = g.DeviceVideo(blobs[c], 6)
    out = torch.empty((1080, 1920, 3), dtype=torch.float32, device="cuda")
    v.render(0, cam, out=out, stats=True)
    for t in range(1, 4):
        v.render_async(t, cs, out)
    v.session.sync()
    v.close()
print("done")
