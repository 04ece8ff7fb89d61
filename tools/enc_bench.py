"""Encoder throughput (dev tool / SURVEY 8(f) row 1): one config-2 group
(300k Gaussians, 30 frames, 6 layers, SH degree 1) held in host memory,
encoded to codec 0+1 by the host-thread encoder and by the GPU encoder; the
two containers must be byte-identical.  Prints one JSON line."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2509_17513_b200.api import Session
from paper_2509_17513_b200.encode import EncodeConfig, encode_stream
from paper_2509_17513_b200.synth import benchmark_spec, iter_frames

n = int(os.environ.get("ENC_N", "300000"))
frames = int(os.environ.get("ENC_FRAMES", "30"))
spec = benchmark_spec(n, frames, int(os.environ.get("ENC_GROUP", "30")))
t0 = time.time()
fr = list(iter_frames(spec, 1002))
gen = time.time() - t0
pos = [f.positions for f in fr]
cfg = EncodeConfig(layer_count=6, prune_fraction=0.0, motion_threshold=0.0025)
sess = Session()
res = {"gaussians": n, "frames": frames, "generate_s": round(gen, 2), "host_threads": os.cpu_count()}
arms = (("gpu", {"device": sess}), ("gpu_warm", {"device": sess}), ("host", {}))
if os.environ.get("ENC_SKIP_HOST"):
    arms = arms[:1]
for name, kw in arms:
    t0 = time.time()
    out = encode_stream(lambda: iter(fr), cfg, codecs=(0, 1), positions_source=lambda: iter(pos), **kw)
    dt = time.time() - t0
    res[name] = {"s": round(dt, 3), "frames_per_s": round(frames / dt, 1),
                 "bytes_c1": len(out[1])}
    res.setdefault("sha", set()).add(hash((out[0], out[1])))
res["identical"] = len(res.pop("sha")) == 1
print(json.dumps(res))
