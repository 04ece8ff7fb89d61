"""ncu driver at full config-2 scale (dev tool): open the whole 300-frame
container (10 groups, resident in HBM) with codec 0 or 1, then render a few
1080p frames.  `python tools/ncu_c2.py 1` -> one rc_decode_kernel launch over
all 1380 runs of the sequence, the launch the bench times."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
import paper_2509_17513_b200 as g
from paper_2509_17513_b200 import _lib


class A:
    gaussians, layers, frames, group, width, height = 300_000, 6, 300, 30, 1920, 1080


codec = int(sys.argv[1]) if len(sys.argv) > 1 else 1
opens = int(sys.argv[2]) if len(sys.argv) > 2 else 1
blobs, _ = bench.make_inputs(A, 1002)
data = blobs[codec]
res = torch.empty(len(data) + 64, dtype=torch.uint8, device="cuda")
res[:len(data)].copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
cam = bench.camera(A)
cs = _lib.camera_struct(cam)
info = g.read_structure(data)
for _ in range(opens):
    v = g.DeviceVideo(data, 6, resident=res, info=info)
    out = torch.empty((1080, 1920, 3), dtype=torch.float32, device="cuda")
    v.render(0, cam, out=out, stats=True)
    for t in range(1, 4):
        v.render_async(t, cs, out)
    v.session.sync()
    v.close()
print("done")
