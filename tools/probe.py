"""Quick performance probe: c2-like scene, stage timings (dev tool)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2509_17513_b200 as g
from paper_2509_17513_b200.encode import EncodeConfig, encode_stream
from paper_2509_17513_b200.synth import benchmark_spec, iter_frames

N = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
F = int(sys.argv[2]) if len(sys.argv) > 2 else 30
t0 = time.time()
spec = benchmark_spec(N, F, 30)
blobs = encode_stream(lambda: iter_frames(spec, 1002), EncodeConfig(layer_count=6, prune_fraction=0.0), codecs=(0, 1))
print(f"encode {time.time()-t0:.1f}s sizes", {k: len(v) for k, v in blobs.items()}, flush=True)
cam = g.Camera.looking_at(eye=(0, 0, -2.5), target=(0, 0, 0), width=1920, height=1080)
for codec in (0, 1):
    for k in (1, 6):
        data = blobs[codec]
        torch.cuda.synchronize()
        t0 = time.time()
        v = g.DeviceVideo(data, k)
        torch.cuda.synchronize()
        t_open = time.time() - t0
        img, st = v.render(0, cam, stats=True)
        s = v.session.stream
        out = torch.empty((1080, 1920, 3), dtype=torch.float32, device="cuda")
        from paper_2509_17513_b200._lib import camera_struct
        cs = camera_struct(cam)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        for t in range(min(3, v.frame_count)):
            v.render_async(t, cs, out)
        e0.record(s)
        for t in range(v.frame_count):
            v.render_async(t, cs, out)
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / v.frame_count
        print(f"codec {codec} k {k}: open {t_open*1e3:.1f} ms (host incl. H2D) | render {ms:.3f} ms/frame | stats {st}", flush=True)
        v.close()
