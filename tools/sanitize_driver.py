"""compute-sanitizer target: smoke() plus one config-1 frame
through every kernel family -- GPU encode (quantise + range code + CRC),
container open (CRC, range decode of both codecs), PlaneLoader projection,
depth sort + tie fix-up, round-1 binning, round-2 emit + tile sort, the
compositor, psnr/ssim, the motion fold, render(list[Splat2D]).

usage: compute-sanitizer --tool memcheck python tools/sanitize_driver.py"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np
import torch

import __graft_entry__ as ge

ge.smoke()

import paper_2509_17513_b200 as g
from paper_2509_17513_b200.configs import CONFIGS, axis_camera, oblique_camera
from paper_2509_17513_b200.encode import EncodeConfig, encode_stream
from paper_2509_17513_b200.synth import iter_frames

c = CONFIGS["c1"]
spec = c.spec()
enc = EncodeConfig(layer_count=c.layers, prune_fraction=0.0)
blobs = encode_stream(lambda: iter_frames(spec, c.seed), enc, codecs=(0, 1), device=True)
for codec in (0, 1):
    with g.DeviceVideo(blobs[codec], c.layers) as v:
        for cam in (axis_camera(c.width, c.height), oblique_camera(c.width, c.height)):
            img = v.render(0, cam)
            img2 = v.render(v.frame_count - 1, cam)
            print("codec", codec, "psnr", g.psnr(img.cpu().numpy().astype(np.float64),
                                                img2.cpu().numpy().astype(np.float64)))
torch.cuda.synchronize()
print("sanitize driver ok")
