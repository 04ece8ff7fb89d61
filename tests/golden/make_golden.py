"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Runs only in the dev container, where /root/reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Everything this writes is data produced by the reference package `gsv`
(/root/reference/pkg/src/gsv): its own conformance fixtures
(pkg/conformance/*.json, copied verbatim), containers encoded by
`encode_sequence`, decoded values from `read_layers`, projection outputs
from `project_set`, images from `render_set` / `render_progressive`, and the
exception class + message the reference raises on corrupted inputs.  The
fixtures travel with the repo; the GPU box never reads /root/reference.
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import shutil
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("GSV_REFERENCE", "/root/reference/pkg"))
sys.path.insert(0, str(REF / "src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from gsv import errors as gerr  # noqa: E402
from gsv.codec import CodecId  # noqa: E402
from gsv.container import read_container_info, read_layers  # noqa: E402
from gsv.gaussians import partition_layers  # noqa: E402
from gsv.motion import frame_delta_between, reconstruct_frame  # noqa: E402
from gsv.pipeline import EncodeConfig, encode_sequence  # noqa: E402
from gsv.render import (Camera, _composite_arrays, project_set, render_progressive,  # noqa: E402
                        render_set)
from gsv.synth import SceneSpec, gen_synthetic_scene  # noqa: E402

OUT = Path(__file__).resolve().parent
TMP = Path("/tmp/golden_work")


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def set_sha(g) -> str:
    return sha(g.positions, g.rotations, g.scales, g.opacities, g.sh)


def cams(width, height):
    return {
        "axis": Camera.looking_at(eye=(0, 0, -2.5), target=(0, 0, 0), fov_deg=60.0,
                                  width=width, height=height, near=0.01),
        "oblique": Camera.looking_at(eye=(1.3, 0.9, -1.9), target=(0, 0, 0), fov_deg=60.0,
                                     width=width, height=height, near=0.01,
                                     background=(0.1, 0.2, 0.3)),
    }


# Synthetic sequence recipes; `scale_k` scales the scale_range
# like (300k/N)^(1/3) so that small scenes still cover the image.
def amps(frames, bursts, base=0.001, burst=0.005):
    """Per-transition translation amplitude with bursts (2 tau_mu) at the
    transitions into `bursts` frames, which forces new groups."""
    return tuple(burst if (a + 1) in bursts else base for a in range(frames - 1))


SCENES = {
    "s1_rc": dict(spec=dict(count=240, frames=6, sh_degree=1, amplitude=amps(6, (3,)),
                            rotation_amplitude=0.01, scale_amplitude=0.0003,
                            opacity_amplitude=0.008, sh_amplitude=0.003,
                            scale_range=(0.03, 0.12), redirect_frames=(3,)),
                  seed=1001, cfg=dict(layer_count=3, codec=1), image=(64, 48)),
    "s1_raw": dict(spec=dict(count=240, frames=6, sh_degree=1, amplitude=amps(6, (3,)),
                             rotation_amplitude=0.01, scale_amplitude=0.0003,
                             opacity_amplitude=0.008, sh_amplitude=0.003,
                             scale_range=(0.03, 0.12), redirect_frames=(3,)),
                   seed=1001, cfg=dict(layer_count=3, codec=0), image=(64, 48)),
    "c1mini_rc": dict(spec=dict(count=1500, frames=4, sh_degree=1, amplitude=amps(4, (2,)),
                                rotation_amplitude=0.01, scale_amplitude=0.0003,
                                opacity_amplitude=0.008, sh_amplitude=0.003,
                                scale_range=(0.02, 0.1), redirect_frames=(2,),
                                ), seed=1001, cfg=dict(layer_count=2, codec=1), image=(96, 64)),
    "deg0_rc": dict(spec=dict(count=64, frames=3, sh_degree=0, amplitude=0.002,
                              rotation_amplitude=0.02, scale_amplitude=0.0004,
                              opacity_amplitude=0.01, sh_amplitude=0.004,
                              scale_range=(0.05, 0.15)), seed=7,
                    cfg=dict(layer_count=2, codec=1, fixed_group_length=2), image=(40, 32)),
    "deg2_rc": dict(spec=dict(count=64, frames=3, sh_degree=2, amplitude=0.002,
                              rotation_amplitude=0.02, scale_amplitude=0.0004,
                              opacity_amplitude=0.01, sh_amplitude=0.004,
                              scale_range=(0.05, 0.15)), seed=8,
                    cfg=dict(layer_count=2, codec=1), image=(40, 32)),
    "deg3_raw": dict(spec=dict(count=64, frames=2, sh_degree=3, amplitude=0.002,
                               rotation_amplitude=0.02, scale_amplitude=0.0004,
                               opacity_amplitude=0.01, sh_amplitude=0.004,
                               scale_range=(0.05, 0.15)), seed=9,
                     cfg=dict(layer_count=3, codec=0), image=(40, 32)),
    "wide32_rc": dict(spec=dict(count=50, frames=3, sh_degree=1, amplitude=0.5,
                                rotation_amplitude=0.02, scale_amplitude=0.0004,
                                opacity_amplitude=0.01, sh_amplitude=0.004,
                                position_extent=120.0, scale_range=(0.5, 2.0)), seed=10,
                      cfg=dict(layer_count=2, codec=1, fixed_group_length=3), image=(40, 32)),
    # the reference's own stream fixture recipe (scripts/make_conformance_fixtures.py:55-99)
    "stream60": dict(spec=dict(count=60, frames=4, sh_degree=1, amplitude=0.001,
                               rotation_amplitude=0.01, scale_amplitude=0.0004,
                               opacity_amplitude=0.01, sh_amplitude=0.004), seed=99,
                     cfg=dict(layer_count=6, codec=1, fixed_group_length=2), image=(40, 32)),
}


def encode(name, rec):
    spec = SceneSpec(**rec["spec"])
    frames = gen_synthetic_scene(spec, rec["seed"])
    c = dict(rec["cfg"])
    cfg = EncodeConfig(layer_count=c["layer_count"], prune_fraction=0.0,
                       motion_threshold=0.0025, codec=CodecId(c["codec"]),
                       fixed_group_length=c.get("fixed_group_length"))
    TMP.mkdir(parents=True, exist_ok=True)
    path = TMP / f"{name}.gsv"
    res = encode_sequence(frames, cfg, path, manifest_path=TMP / f"{name}.manifest.json",
                          keep_reference=True)
    return frames, path.read_bytes(), res


def make_scene(name, rec, doc):
    frames, blob, res = encode(name, rec)
    (OUT / "containers").mkdir(exist_ok=True)
    (OUT / "containers" / f"{name}.gsv").write_bytes(blob)
    info = read_container_info(TMP / f"{name}.gsv")
    L = info.layer_count
    entry = {"recipe": rec, "file_sha256": hashlib.sha256(blob).hexdigest(),
             "layer_count": L, "sh_degree": info.sh_degree,
             "groups": [{"start": g.start_frame, "frames": g.frame_count,
                         "layer_counts": list(g.layer_counts)} for g in info.groups],
             "decode": {}, "renders": {}}
    W, H = rec["image"]
    arrays = {}
    for k in range(1, L + 1):
        video = read_layers(TMP / f"{name}.gsv", k)
        entry["decode"][str(k)] = [set_sha(video.frame(t)) for t in range(video.frame_count)]
        for t in sorted({0, video.frame_count - 1}):
            g = video.frame(t)
            for cname, cam in cams(W, H).items():
                key = f"k{k}_t{t}_{cname}"
                means, covs, depth, colors, opac, rects, idx = project_set(g, cam)
                order = np.argsort(depth, kind="stable")
                img = render_set(g, cam)
                arrays[f"{key}_img"] = img.pixels
                arrays[f"{key}_rects"] = rects
                arrays[f"{key}_idx"] = idx
                arrays[f"{key}_order"] = order
                arrays[f"{key}_depth"] = depth
                arrays[f"{key}_means"] = means
                arrays[f"{key}_cov"] = covs
                arrays[f"{key}_colors"] = colors
                entry["renders"][key] = {"k": k, "t": t, "cam": cname}
    np.savez_compressed(OUT / "renders" / f"{name}.npz", **arrays)
    # full fp64 values for frame 0 at full depth (bit-exact payload check)
    video = read_layers(TMP / f"{name}.gsv", L)
    f0 = video.frame(0)
    np.savez_compressed(OUT / "renders" / f"{name}_frame0.npz", positions=f0.positions,
                        rotations=f0.rotations, scales=f0.scales, opacities=f0.opacities,
                        sh=f0.sh)
    doc[name] = entry
    return blob, info


def cam_json(cam):
    return cam.to_json_dict()


def make_errors(doc):
    """Corrupt containers and record what the reference raises."""
    blob = (OUT / "containers" / "s1_rc.gsv").read_bytes()
    info = read_container_info(TMP / "s1_rc.gsv")
    cases = []

    def probe(name, data, k):
        p = TMP / f"err_{name}.gsv"
        p.write_bytes(data)
        try:
            read_layers(p, k)
        except gerr.GsvError as e:
            return type(e).__name__, str(e)
        return None, None

    # payload bit flips at several places (CRC / structure failures)
    rng = np.random.default_rng(5)
    for gi, g in enumerate(info.groups):
        for layer in range(info.layer_count):
            for ci in (0, 4, len(g.channels[layer]) - 1):
                e = g.channels[layer][ci]
                off = int(e.offset + rng.integers(14, max(15, e.size - 4)))
                bit = int(rng.integers(0, 8))
                data = bytearray(blob)
                data[off] ^= 1 << bit
                for k in (layer + 1, info.layer_count):
                    cls, msg = probe(f"{gi}_{layer}_{ci}", bytes(data), k)
                    cases.append({"kind": "flip", "offset": off, "bit": bit, "k": k,
                                  "error": cls, "message": msg})
    # header / directory damage
    for off, bit in ((0, 0), (4, 1), (6, 0)):
        data = bytearray(blob)
        data[off] ^= 1 << bit
        cls, msg = probe(f"hdr{off}", bytes(data), 1)
        cases.append({"kind": "flip", "offset": off, "bit": bit, "k": 1, "error": cls,
                      "message": msg})
    # truncation
    for cut in (20, 100, len(blob) - 7):
        cls, msg = probe(f"cut{cut}", blob[:cut], info.layer_count)
        cases.append({"kind": "truncate", "length": cut, "k": info.layer_count,
                      "error": cls, "message": msg})
    # layer out of range
    for k in (0, info.layer_count + 1):
        cls, msg = probe(f"k{k}", blob, k)
        cases.append({"kind": "layer", "k": k, "error": cls, "message": msg})
    doc["errors"] = {"container": "s1_rc", "cases": cases}


class _Delta:
    pass


def make_progressive(doc):
    """render_progressive / reconstruct_frame on the reference's moving_scene
    fixture recipe (pkg/tests/conftest.py:34-41, test_render.py:155-178)."""
    spec = SceneSpec(count=90, frames=5, sh_degree=1, amplitude=0.002,
                     rotation_amplitude=0.02, scale_amplitude=0.0004,
                     opacity_amplitude=0.01, sh_amplitude=0.004)
    frames = gen_synthetic_scene(spec, seed=5)
    layered = partition_layers(frames[0], 3, [0.3, 0.3, 0.4], 1e5)
    flat = layered.flatten()
    lookup = {tuple(row): i for i, row in enumerate(frames[0].positions)}
    order = np.array([lookup[tuple(row)] for row in flat.positions], dtype=np.int64)
    deltas = []
    prev = flat
    for t in range(1, 5):
        cur = frames[t].take(order)
        deltas.append(frame_delta_between(prev, cur, t))
        prev = cur
    arrays = {}
    for li, layer in enumerate(layered.layers):
        for nm in ("positions", "rotations", "scales", "opacities", "sh"):
            arrays[f"layer{li}_{nm}"] = getattr(layer, nm)
    for di, d in enumerate(deltas):
        arrays[f"delta{di}_translations"] = d.rigid.translations
        arrays[f"delta{di}_rotations"] = d.rigid.rotations
        arrays[f"delta{di}_d_scales"] = d.residual.d_scales
        arrays[f"delta{di}_d_opacity"] = d.residual.d_opacity
        arrays[f"delta{di}_d_sh"] = d.residual.d_sh
    cam = Camera.looking_at(eye=(0, 0, -2.0), target=(0, 0, 0), width=40, height=40)
    out = {"layer_count": 3, "n_deltas": len(deltas), "sh_degree": 1,
           "camera": cam_json(cam), "cases": {}}
    for k in (1, 2, 3):
        for t in (0, 1, 2, 4):
            g = reconstruct_frame(layered, deltas, t, up_to_layer=k)
            key = f"k{k}_t{t}"
            for nm in ("positions", "rotations", "scales", "opacities", "sh"):
                arrays[f"recon_{key}_{nm}"] = getattr(g, nm)
            arrays[f"img_{key}"] = render_progressive(layered, k, deltas, t, cam).pixels
            out["cases"][key] = {"k": k, "t": t}
    np.savez_compressed(OUT / "renders" / "progressive.npz", **arrays)
    doc["progressive"] = out


def make_known_answer(doc):
    """render() known-answer scenes (test_render.py:77-115) and the 10 random
    acceptance scenes at 256^2 (test_acceptance.py:155-169)."""
    from gsv.render import Splat2D, render
    arrays = {}
    cam = Camera(rotation=np.eye(3), translation=np.zeros(3), fx=100.0, fy=100.0,
                 cx=32, cy=32, width=64, height=64, near=0.1)

    def flat(alpha, color, depth):
        return Splat2D(mean2d=np.array([32.0, 32.0]), cov2d=np.eye(2) * 1e6, depth=depth,
                       color=np.full(3, color), base_opacity=alpha)
    arrays["single_opaque"] = render([flat(1.0, 1.0, 1.0)], cam).pixels
    arrays["two_over"] = render([flat(0.5, 1.0, 1.0), flat(1.0, 0.0, 2.0)], cam).pixels
    scenes = []
    for i in range(10):
        spec = SceneSpec(count=300, frames=1, sh_degree=1, scale_range=(0.02, 0.08))
        g = gen_synthetic_scene(spec, seed=300 + i)[0]
        cam2 = Camera.looking_at(eye=(0.2 * i - 1.0, 0.3, -2.2), target=(0, 0, 0),
                                 width=64, height=64)
        arrays[f"accept{i}_img"] = render_set(g, cam2).pixels
        scenes.append({"seed": 300 + i, "camera": cam_json(cam2)})
    np.savez_compressed(OUT / "renders" / "known_answer.npz", **arrays)
    doc["known_answer"] = {"camera": cam_json(cam), "accept": scenes}


def make_render2d(doc):
    """render(list[Splat2D]) on random projected splats (ragged rects at the
    image border, exact depth ties, negative depths, empty rects) and psnr
    values between reference images (metrics.py:31-38)."""
    from gsv.metrics import psnr, ssim
    from gsv.render import Splat2D, render
    rng = np.random.default_rng(4242)
    cam = Camera(rotation=np.eye(3), translation=np.zeros(3), fx=90.0, fy=90.0,
                 cx=40.0, cy=30.0, width=80, height=60, near=0.1, background=(0.1, 0.2, 0.3))
    n = 400
    means = rng.uniform(-10, 90, size=(n, 2))
    sx = rng.uniform(0.3, 6.0, n)
    sy = rng.uniform(0.3, 6.0, n)
    rho = rng.uniform(-0.8, 0.8, n)
    cov = np.stack([np.stack([sx * sx, rho * sx * sy], -1), np.stack([rho * sx * sy, sy * sy], -1)], -2)
    depth = np.round(rng.uniform(-1.0, 3.0, n), 1)  # many exact ties, some negative
    colors = rng.uniform(0, 1, size=(n, 3))
    opac = rng.uniform(0.05, 1.0, n)
    opac[::37] = 0.0
    splats = [Splat2D(mean2d=means[i], cov2d=cov[i], depth=float(depth[i]), color=colors[i],
                      base_opacity=float(opac[i])) for i in range(n)]
    img = render(splats, cam).pixels
    img_half = render(splats[: n // 2], cam).pixels
    arrays = {"means": means, "cov": cov, "depth": depth, "colors": colors, "opac": opac,
              "img": img, "img_half": img_half}
    np.savez_compressed(OUT / "renders" / "render2d.npz", **arrays)
    from gsv.render import Image as RImage
    doc["render2d"] = {"camera": cam_json(cam), "n": n,
                       "psnr_full_half": psnr(RImage(img), RImage(img_half)),
                       "psnr_same": psnr(RImage(img), RImage(img)),
                       "ssim_full_half": ssim(RImage(img), RImage(img_half)),
                       "ssim_same": ssim(RImage(img), RImage(img))}


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--only-render2d":
        doc = json.loads((OUT / "golden.json").read_text())
        make_render2d(doc)
        (OUT / "golden.json").write_text(json.dumps(doc, indent=1, default=float) + "\n")
        return
    if TMP.exists():
        shutil.rmtree(TMP)
    TMP.mkdir(parents=True)
    (OUT / "renders").mkdir(exist_ok=True)
    conf = OUT / "conformance"
    conf.mkdir(exist_ok=True)
    for p in sorted((REF / "conformance").glob("*.json")):
        shutil.copyfile(p, conf / p.name)
    doc = {"scenes": {}}
    for name, rec in SCENES.items():
        make_scene(name, rec, doc["scenes"])
        print("scene", name, "ok", flush=True)
    cam_doc = {}
    for name, rec in SCENES.items():
        W, H = rec["image"]
        cam_doc[name] = {k: cam_json(c) for k, c in cams(W, H).items()}
    doc["cameras"] = cam_doc
    make_errors(doc)
    make_progressive(doc)
    make_known_answer(doc)
    make_render2d(doc)
    (OUT / "golden.json").write_text(json.dumps(doc, indent=1, default=float) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
