"""Driver for ncu captures of the motion warp (fold_kernel: motion.py:165-193
reconstruct_frame on the device; dev tool): a 300k-Gaussian SH-1 keyframe and
29 frame deltas folded to frame 29."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2509_17513_b200 import api
from paper_2509_17513_b200.types import (FrameDelta, GaussianSet, LayeredFrame, ResidualDelta,
                                         RigidDelta)

n, nd = 300_000, 29
rng = np.random.default_rng(5)
q = rng.normal(size=(n, 4))
key = GaussianSet(rng.uniform(-1, 1, (n, 3)), q / np.linalg.norm(q, axis=1, keepdims=True),
                  rng.uniform(0.004, 0.02, (n, 3)), rng.uniform(0.2, 1.0, n), rng.normal(size=(n, 12)), 1)
frame = LayeredFrame(layers=(key,), layer_fractions=(1.0,), volume_weight=1e5)
deltas = []
for f in range(nd):
    dq = np.concatenate([np.ones((n, 1)), rng.normal(scale=1e-3, size=(n, 3))], axis=1)
    dq /= np.linalg.norm(dq, axis=1, keepdims=True)
    deltas.append(FrameDelta(RigidDelta(rng.normal(scale=1e-3, size=(n, 3)), dq),
                             ResidualDelta(rng.normal(scale=1e-4, size=(n, 3)), rng.normal(scale=1e-3, size=n),
                                           rng.normal(scale=1e-3, size=(n, 12))), f + 1))
for _ in range(3):
    api.reconstruct_frame_tensors(frame, deltas, nd)
torch.cuda.synchronize()
print("done")
