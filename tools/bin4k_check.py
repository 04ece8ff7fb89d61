"""Dev check: the round-1 counting placement against emit + sort on a 4K
frame (32400 tiles: 130 KB of shared counters) -- images must be identical."""
import os
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
if len(sys.argv) > 1:  # child: render and save
    import numpy as np
    import torch

    import bench
    import paper_2509_17513_b200 as g

    class A:
        gaussians, layers, frames, group, width, height = 300_000, 6, 30, 30, 3840, 2160
    blobs, _ = bench.make_inputs(A, 1002)
    v = g.DeviceVideo(blobs[0], 6)
    out = [v.render(t, bench.camera(A)).cpu().numpy() for t in (0, 17)]
    np.save(sys.argv[1], np.stack(out))
    sys.exit(0)
for b in (0, 1):
    env = dict(os.environ, GSV_R1_BIN=str(b))
    subprocess.run([sys.executable, __file__, f"/tmp/bin4k_{b}.npy"], env=env, check=True)
import numpy as np
x, y = np.load("/tmp/bin4k_0.npy"), np.load("/tmp/bin4k_1.npy")
print("4K identical:", np.array_equal(x, y), "max diff", float(np.abs(x - y).max()), "mean", float(x.mean()))
