"""Dev A/B of compositor variants (GSV_COMPOSITE_* knobs are read once per
process, so every variant runs in its own subprocess).

    python tools/composite_ab.py VAR=VAL[,VAR=VAL] ...     (one arg per variant; "" = defaults)

Per variant: a config-2 group (300k Gaussians, 6 layers, 30 frames, codec 0,
cached under /tmp) rendered at 1080p for the axis and oblique cameras;
reports frames/s of render_batch (8 streams, 5 reps of 30 frames) and the
max-abs / differing-pixel count of every image against the first variant.
"""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out" / "ab"


def child(tag):
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch

    import paper_2509_17513_b200 as g
    from paper_2509_17513_b200.configs import CONFIGS, axis_camera, oblique_camera
    from paper_2509_17513_b200.encode import EncodeConfig, encode_stream
    from paper_2509_17513_b200.synth import iter_frames

    cache = Path("/tmp/gsv_ab_c2g30.gsv")
    if not cache.exists():
        cfg = CONFIGS["c2"]
        spec = cfg.spec(30)
        enc = EncodeConfig(layer_count=cfg.layers, prune_fraction=0.0, motion_threshold=0.0025)
        blobs = encode_stream(lambda: iter_frames(spec, cfg.seed), enc, codecs=(0,), device=True,
                              positions_source=lambda: iter_frames(spec, cfg.seed, positions_only=True))
        cache.write_bytes(blobs[0])
    data = cache.read_bytes()
    res = {}
    imgs = {}
    with g.DeviceVideo(data, 6) as v:
        for cname, cam in (("axis", axis_camera(1920, 1080)), ("oblique", oblique_camera(1920, 1080))):
            for t in (0, 29):
                imgs[f"{cname}{t}"] = v.render(t, cam).cpu().numpy()
            frames = list(range(30))
            outs = [torch.empty((1080, 1920, 3), dtype=torch.float32, device="cuda") for _ in frames]
            v.render_batch(frames, cam, outs=outs)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                v.render_batch(frames, cam, outs=outs, verify=False)
            torch.cuda.synchronize()
            res[cname] = 150 / (time.perf_counter() - t0)
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez(OUT / f"{tag}.npz", **imgs)
    print(json.dumps(res))


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        return child(sys.argv[2])
    import numpy as np
    variants = sys.argv[1:] or [""]
    base = None
    for i, var in enumerate(variants):
        env = dict(os.environ)
        for kv in filter(None, var.split(",")):
            k, v = kv.split("=", 1)
            env[k] = v
        tag = f"v{i}"
        r = subprocess.run([sys.executable, __file__, "--child", tag], env=env, capture_output=True, text=True)
        if r.returncode:
            print(f"[{var or 'default'}] FAILED\n{r.stderr[-3000:]}")
            continue
        fps = json.loads(r.stdout.strip().splitlines()[-1])
        imgs = dict(np.load(OUT / f"{tag}.npz"))
        diff = ""
        if base is None:
            base = imgs
        else:
            d = [(k, float(np.max(np.abs(imgs[k] - base[k]))), int(np.sum(imgs[k] != base[k]))) for k in imgs]
            diff = " ".join(f"{k}:max{m:.2e}/n{n}" for k, m, n in d)
        print(f"[{var or 'default'}] fps axis {fps['axis']:.0f} oblique {fps['oblique']:.0f} {diff}", flush=True)


if __name__ == "__main__":
    main()
