"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle.

Bars (BASELINE.json north_star): bit-exact for dequantized integer symbols /
fp64 values, group assignment, rects, tile counts and depth order; images
within max-abs 2e-3 per channel and |dPSNR| <= 0.01 dB.
"""

import base64
import json

import numpy as np
import pytest

from golden_util import (GOLDEN, Cam, camera, container, doc, progressive_inputs, renders,
                         scene_names, set_sha)
from oracle import oracle as O

pytestmark = pytest.mark.gpu

MAX_ABS = 2e-3
MAX_DPSNR = 0.01


@pytest.fixture(scope="module")
def gsvb():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2509_17513_b200 as m
    return m


def test_native_library_is_loaded(gsvb):
    from paper_2509_17513_b200 import _lib
    L = _lib.load()
    maps = open("/proc/self/maps").read()
    assert str(_lib.LIB_PATH) in maps


@pytest.mark.parametrize("path", sorted((GOLDEN / "conformance").glob("*.json")),
                         ids=lambda p: p.stem)
def test_conformance_payloads_gpu(gsvb, path):
    d = json.loads(path.read_text())
    blob = base64.b64decode(d["payload_b64"])
    payload, end = gsvb.CodedPayload.from_bytes(blob)
    assert end == len(blob)
    planes = gsvb.decode_planes(payload)
    assert len(planes) == d["count"]
    for plane, exp in zip(planes, d["expected_samples"]):
        assert plane.samples.ravel().tolist() == exp


def test_decode_planes_corruption_gpu(gsvb):
    d = json.loads((GOLDEN / "conformance" / "rc_u8_random.json").read_text())
    blob = bytearray(base64.b64decode(d["payload_b64"]))
    blob[20] ^= 0x04
    payload, _ = gsvb.CodedPayload.from_bytes(bytes(blob))
    with pytest.raises(gsvb.CodecError):
        gsvb.decode_planes(payload)


@pytest.mark.parametrize("name", scene_names())
def test_decode_bit_exact_and_group_assignment(gsvb, name):
    sc = doc()["scenes"][name]
    data = container(name)
    for k in range(1, sc["layer_count"] + 1):
        with gsvb.DeviceVideo(data, k) as v:
            assert v.frame_count == sum(g["frames"] for g in sc["groups"])
            info = O.read_structure(data)
            for t in range(v.frame_count):
                assert v.group_of(t) == O.group_of(info, t)
                assert set_sha(v.frame(t)) == sc["decode"][str(k)][t], (name, k, t)
            # integer symbols against the oracle's decode
            _, _ = O.read_layers(data, k)
            gi = v.group_of(0)
            vals = O.decode_group_codes(data, info, gi, k)
            codes = v.frame_codes(0).cpu().numpy().astype(np.uint32)
            deg = info.sh_degree
            order = [("position", c) for c in range(3)] + [("rotation", c) for c in range(4)] + \
                [("scales", c) for c in range(3)] + [("opacity", 0)] + \
                [("sh", c) for c in range(3 * (deg + 1) ** 2)]
            exp = np.concatenate([np.stack([vals[l][key][0][0] for key in order], axis=1)
                                  for l in range(k)])
            assert np.array_equal(codes, exp)


@pytest.mark.parametrize("name", scene_names())
def test_render_matches_reference_images(gsvb, name):
    sc = doc()["scenes"][name]
    data = container(name)
    arr = renders(name)
    for key, r in sc["renders"].items():
        cam = camera(name, r["cam"])
        with gsvb.DeviceVideo(data, r["k"]) as v:
            img, st = v.render(r["t"], cam, stats=True)
            got = img.cpu().numpy().astype(np.float64)
            g = v.frame(r["t"])
        ref = arr[f"{key}_img"]
        err = float(np.max(np.abs(got - ref)))
        assert err <= MAX_ABS, (key, err)
        # counts are bit-exact: survivors and tile keys from the reference rects
        rects = arr[f"{key}_rects"]
        assert st["n_visible"] == rects.shape[0]
        assert st["n_keys"] == int(O.tile_counts(rects).sum())
        # projection: rects, depth, order, tile counts exact
        prect, pdepth, porder, ptiles, nvis = gsvb.project_debug(g, cam)
        idx = arr[f"{key}_idx"]
        assert nvis == idx.size
        assert np.array_equal(prect[idx].astype(np.int64), rects)
        assert np.array_equal(pdepth[idx], arr[f"{key}_depth"])
        assert np.array_equal(porder[:nvis], idx[arr[f"{key}_order"]])
        assert np.array_equal(ptiles[idx], O.tile_counts(rects))


def test_error_paths_match_reference(gsvb):
    errs = doc()["errors"]
    blob = container(errs["container"])
    classes = {"CodecError": gsvb.CodecError, "FormatError": gsvb.FormatError,
               "InvalidInputError": gsvb.InvalidInputError}
    for case in errs["cases"]:
        data = bytearray(blob)
        if case["kind"] == "flip":
            data[case["offset"]] ^= 1 << case["bit"]
        elif case["kind"] == "truncate":
            data = data[:case["length"]]
        if case["error"] is None:
            gsvb.DeviceVideo(bytes(data), case["k"]).close()
            continue
        with pytest.raises(classes[case["error"]]) as ei:
            gsvb.DeviceVideo(bytes(data), case["k"])
        assert str(ei.value) == case["message"], case


def test_progressive_matches_reference(gsvb):
    layers, deltas, cam, d, a = progressive_inputs()
    frame = gsvb.LayeredFrame(layers=tuple(layers), layer_fractions=(0.3, 0.3, 0.4),
                              volume_weight=1e5)
    for key, c in d["cases"].items():
        g = gsvb.reconstruct_frame(frame, deltas, c["t"], c["k"])
        for nm in ("positions", "rotations", "scales", "opacities", "sh"):
            assert np.array_equal(getattr(g, nm), a[f"recon_{key}_{nm}"]), (key, nm)
        img = gsvb.render_progressive(frame, c["k"], deltas, c["t"], cam)
        assert np.max(np.abs(img.pixels - a[f"img_{key}"])) <= MAX_ABS, key
    with pytest.raises(gsvb.InvalidInputError, match="layer 4 out of range 1..3"):
        gsvb.render_progressive(frame, 4, deltas, 0, cam)


def test_acceptance_scenes(gsvb):
    from paper_2509_17513_b200.synth import SceneSpec, iter_frames
    ka = doc()["known_answer"]
    arr = renders("known_answer")
    for i, sc in enumerate(ka["accept"]):
        g = next(iter_frames(SceneSpec(count=300, frames=1, sh_degree=1,
                                       scale_range=(0.02, 0.08)), sc["seed"]))
        cam = Cam.from_json(sc["camera"])
        img = gsvb.render_set(g, cam)
        assert np.max(np.abs(img.pixels - arr[f"accept{i}_img"])) <= MAX_ABS


def _bench_scene(count, frames, group_len, layers, codec, seed):
    from paper_2509_17513_b200.encode import EncodeConfig, encode_stream
    from paper_2509_17513_b200.synth import benchmark_spec, iter_frames
    spec = benchmark_spec(count, frames, group_len)
    cfg = EncodeConfig(layer_count=layers, prune_fraction=0.0, codec=codec)
    return encode_stream(lambda: iter_frames(spec, seed), cfg, codecs=(0, 1)), spec


def _psnr(a, b):
    return O.psnr(a, b)


def test_config1_full_parity(gsvb):
    """BASELINE config 1: 50k Gaussians, 2 layers, 4 frames (2 groups), 512^2,
    both codecs, every frame and prefix, axis + oblique cameras."""
    from paper_2509_17513_b200.synth import benchmark_spec, iter_frames
    blobs, spec = _bench_scene(50_000, 4, 2, 2, 1, 1001)
    assert blobs[0] != blobs[1]
    frames_src = list(iter_frames(spec, 1001))
    for cname, cam in (("axis", Cam.from_json(_cam_json(512, 512, (0, 0, -2.5)))),
                       ("oblique", Cam.from_json(_cam_json(512, 512, (1.3, 0.9, -1.9))))):
        for codec in (0, 1):
            data = blobs[codec]
            for k in (1, 2):
                _, groups = O.read_layers(data, k)
                with gsvb.DeviceVideo(data, k) as v:
                    for t in range(4):
                        g = O.frame_of(groups, t)
                        img = v.render(t, cam).cpu().numpy().astype(np.float64)
                        ref = O.render_set(g, cam)
                        assert np.max(np.abs(img - ref)) <= MAX_ABS, (codec, k, t, cname)
                        if codec == 1 and k == 2:
                            gt = O.render_set(frames_src[t], cam)
                            assert abs(_psnr(gt, img) - _psnr(gt, ref)) <= MAX_DPSNR


def _cam_json(w, h, eye):
    from paper_2509_17513_b200.types import Camera
    return Camera.looking_at(eye=eye, target=(0, 0, 0), fov_deg=60.0, width=w, height=h,
                             near=0.01).to_json_dict()


def test_config2_frame_parity(gsvb):
    """BASELINE config 2 geometry: 300k Gaussians, 6 layers, 1080p; two frames
    (one group) checked against the oracle at k = 1 and 6."""
    blobs, spec = _bench_scene(300_000, 2, 30, 6, 1, 1002)
    cam = Cam.from_json(_cam_json(1920, 1080, (0, 0, -2.5)))
    data = blobs[1]
    for k in (1, 6):
        _, groups = O.read_layers(data, k)
        with gsvb.DeviceVideo(data, k) as v:
            for t in (0, 1):
                g = O.frame_of(groups, t)
                img, st = v.render(t, cam, stats=True)
                img = img.cpu().numpy().astype(np.float64)
                means, covs, depth, colors, opac, rects, idx = O.project_set(g, cam)
                ref = O.composite(means, covs, depth, colors, opac, rects, cam)
                assert st["n_visible"] == idx.size
                assert st["n_keys"] == int(O.tile_counts(rects).sum())
                assert np.max(np.abs(img - ref)) <= MAX_ABS, (k, t)


@pytest.mark.gpu
def test_render2d_and_psnr_gpu(gsvb):
    """render(list[Splat2D]) on the GPU vs the reference image (stable depth
    order with exact ties and negative depths, border-clipped and empty
    rects, zero opacities): max-abs <= 2e-3; psnr on the GPU vs the
    reference's value |dPSNR| <= 0.01 dB."""
    from golden_util import Cam, doc, renders
    d = doc()["render2d"]
    r = renders("render2d")
    cam = Cam.from_json(d["camera"])
    splats = [gsvb.Splat2D(mean2d=r["means"][i], cov2d=r["cov"][i], depth=float(r["depth"][i]),
                           color=r["colors"][i], base_opacity=float(r["opac"][i]))
              for i in range(len(r["depth"]))]
    img = gsvb.render(splats, cam).pixels
    assert np.max(np.abs(img - r["img"])) <= 2e-3
    half = gsvb.render(splats[: len(splats) // 2], cam).pixels
    assert np.max(np.abs(half - r["img_half"])) <= 2e-3
    assert abs(gsvb.psnr(img, half) - d["psnr_full_half"]) <= 0.01
    assert abs(gsvb.psnr(gsvb.Image(r["img"]), gsvb.Image(r["img_half"])) - d["psnr_full_half"]) <= 1e-9
    assert gsvb.psnr(img, img) == 99.0
    bg = gsvb.render([], cam).pixels
    assert np.array_equal(bg, np.tile(np.asarray(cam.background), (cam.height, cam.width, 1)))


@pytest.mark.gpu
def test_ssim_gpu(gsvb):
    """ssim on the GPU (separable 11x11 Gaussian window, fp64) vs the
    reference's scipy convolve2d value, fp64 and fp32 inputs."""
    import torch
    from golden_util import doc, renders
    d = doc()["render2d"]
    r = renders("render2d")
    assert abs(gsvb.ssim(r["img"], r["img_half"]) - d["ssim_full_half"]) <= 1e-9
    assert abs(gsvb.ssim(gsvb.Image(r["img"]), gsvb.Image(r["img"])) - 1.0) <= 1e-12
    f32 = gsvb.ssim(torch.from_numpy(r["img"]).float().cuda(), torch.from_numpy(r["img_half"]).float().cuda())
    assert abs(f32 - d["ssim_full_half"]) <= 1e-5
    assert abs(gsvb.d_ssim(r["img"], r["img_half"]) - (1 - d["ssim_full_half"]) / 2) <= 1e-9
    with pytest.raises(gsvb.InvalidInputError):
        gsvb.ssim(np.zeros((8, 8, 3)), np.zeros((8, 8, 3)))


@pytest.mark.gpu
def test_analyze_rd_gpu(gsvb, tmp_path):
    """cmd_analyze's loop (cli.py:147-162) on the GPU: decode at a layer
    prefix, render every frame, PSNR against ground truth on the device; the
    mean PSNR per container matches the CPU oracle's within 0.01 dB and the
    rate is the layer-prefix payload per frame."""
    name = "s1_rc"
    data = container(name)
    p = tmp_path / "c.gsv"
    p.write_bytes(data)
    cam = camera(name, "oblique")
    L = doc()["scenes"][name]["layer_count"]
    _, gt_groups = O.read_layers(data, L)
    nfr = sum(g.frame_count for g in O.read_structure(data).groups)
    gts = [O.render_set(O.frame_of(gt_groups, t), cam) for t in range(nfr)]
    for k in (1, L):
        (rate, mean_psnr), = gsvb.analyze_rd([str(p)], cam, gts, layer=k)
        _, groups = O.read_layers(data, k)
        ref = float(np.mean([O.psnr(gts[t], O.render_set(O.frame_of(groups, t), cam)) for t in range(nfr)]))
        assert abs(mean_psnr - ref) <= 0.01, (k, mean_psnr, ref)
        info = O.read_structure(data)
        payload = sum(e.size for g in info.groups for l in range(k) for e in g.channels[l])
        assert rate == payload / nfr / 1e6


@pytest.mark.gpu
def test_open_group_range(gsvb):
    """gsv_video_open_groups: a group range decodes exactly like those groups
    of the whole container (frames numbered from 0 in the range)."""
    name = "s1_rc"
    data = container(name)
    info = O.read_structure(data)
    G = len(info.groups)
    assert G >= 2
    k = doc()["scenes"][name]["layer_count"]
    _, groups = O.read_layers(data, k)
    start = 0
    for g in range(G):
        with gsvb.DeviceVideo(data, k, groups=(g, g + 1)) as v:
            assert v.frame_count == info.groups[g].frame_count
            for i in range(v.frame_count):
                got, ref = v.frame(i), O.frame_of(groups, start + i)
                for nm in ("positions", "rotations", "scales", "opacities", "sh"):
                    assert np.array_equal(getattr(got, nm), getattr(ref, nm)), (g, i, nm)
        start += info.groups[g].frame_count
    with pytest.raises(gsvb.InvalidInputError):
        gsvb.DeviceVideo(data, k, groups=(G, G + 1))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["huge_splats", "tiny_image", "behind_camera", "many_rounds"])
def test_render_edge_cases(gsvb, case):
    """Edge cases of the tiled compositor against the oracle: splats that
    cover the whole image (key buffers grow and re-render), an image smaller
    than one tile (partial tiles on both axes), every splat culled (pure
    background), and more splats than the first depth-rank round holds (open
    tiles carried into a second round)."""
    from paper_2509_17513_b200.synth import SceneSpec, iter_frames
    from paper_2509_17513_b200.types import Camera
    if case == "huge_splats":
        spec, W, H, eye = SceneSpec(count=2000, frames=1, sh_degree=1, scale_range=(0.3, 0.9)), 160, 120, (0, 0, -2.5)
    elif case == "tiny_image":
        spec, W, H, eye = SceneSpec(count=500, frames=1, sh_degree=2, scale_range=(0.02, 0.1)), 13, 9, (0.4, 0.2, -2.4)
    elif case == "behind_camera":
        spec, W, H, eye = SceneSpec(count=500, frames=1, sh_degree=0, scale_range=(0.02, 0.1)), 64, 48, (0, 0, 5.0)
    else:
        spec, W, H, eye = SceneSpec(count=40_000, frames=1, sh_degree=1, scale_range=(0.004, 0.03)), 320, 240, (0.3, -0.2, -2.5)
    g = next(iter(iter_frames(spec, 777)))
    cam = Camera.looking_at(eye=eye, target=(0, 0, 0.0 if case != "behind_camera" else 10.0),
                            fov_deg=60.0, width=W, height=H, near=0.01,
                            background=(0.2, 0.1, 0.05))
    img = gsvb.render_set(g, cam).pixels
    ref = O.render_set(g, cam)
    assert img.shape == (H, W, 3)
    assert np.max(np.abs(img - ref)) <= MAX_ABS, case
    if case == "behind_camera":
        assert np.array_equal(img, np.tile(np.asarray(cam.background, np.float64), (H, W, 1)).astype(np.float32))


_PATHS_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
import paper_2509_17513_b200 as g
from golden_util import camera, container
out = []
for name in ('s1_rc', 'c1mini_rc'):
    data = container(name)
    with g.DeviceVideo(data, None) as v:
        for which in ('axis', 'oblique'):
            cam = camera(name, which)
            for t in (0, v.frame_count - 1):
                out.append(v.render(t, cam).cpu().numpy())
np.save(sys.argv[2], np.stack([o.ravel() for o in out]) if len({o.size for o in out}) == 1
        else np.concatenate([o.ravel() for o in out]))
"""


def test_binning_and_sort_paths_render_identically(tmp_path):
    """The round-1 counting placement and the round-2 tile ranges against the
    emit + sort + key-search path they replace (GSV_R1_BIN=0 GSV_R2_RANGES=0,
    also the path of frames above 32768 tiles): bit-identical images."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    for tag, env in (("fast", {}), ("sort", {"GSV_R1_BIN": "0", "GSV_R2_RANGES": "0"})):
        f = tmp_path / f"{tag}.npy"
        subprocess.run([sys.executable, "-c", _PATHS_SCRIPT, root, str(f)], check=True,
                       env={**os.environ, **env}, timeout=600)
        res[tag] = np.load(f)
    assert np.array_equal(res["fast"], res["sort"])


def test_compositor_variants_render_identically(tmp_path):
    """Compositor V2 (per-lane record terms), V3 (staged quad, full-height
    records without the vote) and V4 (the default: per-column tables) compute
    the same operations: bit-identical images (GSV_COMPOSITE_PACKED=2/3/4)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    for tag in ("2", "3", "4"):
        f = tmp_path / f"v{tag}.npy"
        subprocess.run([sys.executable, "-c", _PATHS_SCRIPT, root, str(f)], check=True,
                       env={**os.environ, "GSV_COMPOSITE_PACKED": tag}, timeout=600)
        res[tag] = np.load(f)
    assert np.array_equal(res["2"], res["3"])
    assert np.array_equal(res["3"], res["4"])


@pytest.mark.parametrize("bits", [8, 16])
def test_truncated_coded_block_is_codec_error(gsvb, bits):
    """A range-coded plane whose coded block is far shorter than the plane
    needs (4 bytes for 4M samples): the decoder zero-fills past the block
    like the reference (_rc.py:129,150) without reading past it, and the CRC
    mismatch raises CodecError -- no illegal address, the context stays
    usable."""
    import struct
    w = h = 2048
    block = bytes([0x00, 0x9C, 0x41, 0x07])
    body = bytes([0, 0]) + struct.pack("<I", len(block)) + block
    blob = struct.pack("<BBHHHHI", 1, bits, w, h, 1, 0, len(body)) + body + struct.pack("<I", 0x12345678)
    payload, end = gsvb.CodedPayload.from_bytes(blob)
    assert end == len(blob)
    with pytest.raises(gsvb.CodecError, match="checksum mismatch"):
        gsvb.decode_planes(payload)
    # the device is still healthy: a good payload decodes afterwards
    d = json.loads((GOLDEN / "conformance" / "rc_u8_random.json").read_text())
    good, _ = gsvb.CodedPayload.from_bytes(base64.b64decode(d["payload_b64"]))
    assert gsvb.decode_planes(good)[0].samples.ravel().tolist() == d["expected_samples"][0]


@pytest.mark.parametrize("variant", ["1", "2", "3", "4", "5", "6"])
def test_range_decoder_variants_bit_exact(gsvb, variant, monkeypatch):
    """Every range-decoder variant (GSV_RC_VARIANT: 1 C++ fast path, 2 PTX
    step, 3 + zero-prefix test, 4 + saturated zero-prefix test, 5 warp-
    cooperative speculation, the default)
    decodes the reference-encoded codec-1 containers to the oracle's integer
    codes at every frame."""
    monkeypatch.setenv("GSV_RC_VARIANT", variant)
    for name in ("c1mini_rc", "s1_rc", "deg2_rc", "wide32_rc"):
        data = container(name)
        info = O.read_structure(data)
        k = info.layer_count
        deg = info.sh_degree
        order = [("position", c) for c in range(3)] + [("rotation", c) for c in range(4)] + \
            [("scales", c) for c in range(3)] + [("opacity", 0)] + \
            [("sh", c) for c in range(3 * (deg + 1) ** 2)]
        with gsvb.DeviceVideo(data, k) as v:
            for t in range(v.frame_count):
                gi = v.group_of(t)
                vals = O.decode_group_codes(data, info, gi, k)
                tl = t - info.groups[gi].start_frame
                exp = np.concatenate([np.stack([vals[l][key][0][tl] for key in order], axis=1)
                                      for l in range(k)])
                got = v.frame_codes(t).cpu().numpy().astype(np.uint32)
                assert np.array_equal(got, exp), (name, t)
