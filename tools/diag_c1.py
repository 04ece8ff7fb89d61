"""Dev diagnostic: config-1 render error vs the CPU oracle (packed / scalar compositor)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent)); sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
import paper_2509_17513_b200 as gsvb
from oracle import oracle as O
from test_gpu_parity import _bench_scene, _cam_json, _psnr
from golden_util import Cam
from paper_2509_17513_b200.synth import iter_frames
blobs, spec = _bench_scene(50_000, 4, 2, 2, 1, 1001)
frames_src = list(iter_frames(spec, 1001))
for cname, eye in (("axis", (0, 0, -2.5)), ("oblique", (1.3, 0.9, -1.9))):
    cam = Cam.from_json(_cam_json(512, 512, eye))
    data = blobs[1]
    _, groups = O.read_layers(data, 2)
    with gsvb.DeviceVideo(data, 2) as v:
        for t in range(2):
            g = O.frame_of(groups, t)
            img = v.render(t, cam).cpu().numpy().astype(np.float64)
            ref = O.render_set(g, cam)
            err = np.abs(img - ref)
            i = np.unravel_index(err.argmax(), err.shape)
            gt = O.render_set(frames_src[t], cam)
            print(cname, t, "maxabs", err.max(), "at", i, "ref", ref[i[0], i[1]], "gpu", img[i[0], i[1]],
                  "n>1e-3", int((err > 1e-3).sum()), "dpsnr", _psnr(gt, img) - _psnr(gt, ref), flush=True)
