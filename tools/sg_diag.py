"""Dev diagnostic: open vs render time for the 2-frame-group container."""
import sys, time, copy
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
import paper_2509_17513_b200 as gsvb
from paper_2509_17513_b200 import _lib
class A:
    gaussians, layers, frames, group, width, height, k, streams = 300_000, 6, 300, 2, 1920, 1080, 6, 8
a = A()
blobs, _ = bench.make_inputs(a, 1003)
cs = _lib.camera_struct(bench.camera(a))
sess = gsvb.Session(0)
outs = [torch.empty((1080, 1920, 3), dtype=torch.float32, device="cuda") for _ in range(300)]
for codec in (0, 1):
    data = blobs[codec]
    dev = torch.empty(len(data) + 64, dtype=torch.uint8, device="cuda"); dev[:len(data)].copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
    info = gsvb.read_structure(data)
    for it in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        v = gsvb.DeviceVideo(data, 6, session=sess, resident=dev, info=info)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        v.render_batch(list(range(300)), cs, outs=outs, streams=8, verify=(it == 0))
        torch.cuda.synchronize(); t2 = time.perf_counter()
        _, st = v.render(0, bench.camera(a), stats=True)
        v.close()
        print(f"codec{codec} open {1e3*(t1-t0):.1f} ms render {1e3*(t2-t1):.1f} ms stats {st}", flush=True)
