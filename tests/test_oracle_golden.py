"""Pin the CPU oracle (oracle/) to the reference's golden vectors.

Every fixture was produced by the real reference (tests/golden/make_golden.py).
Integer work (samples, codes, rects, order, group assignment) and fp64
decode/projection values must match bit-exactly; composited images to 1e-12
(the only difference allowed is libm exp vs numba's).
"""

import base64
import json
from pathlib import Path

import numpy as np
import pytest

from golden_util import (GOLDEN, camera, container, doc, progressive_inputs, renders,
                         scene_names, set_sha)
from oracle import oracle as O

CONF = sorted((GOLDEN / "conformance").glob("*.json"))


def test_conformance_fixtures_present():
    assert len(CONF) >= 7


@pytest.mark.parametrize("path", CONF, ids=lambda p: p.stem)
def test_conformance_payloads(path):
    """test_conformance.py:25-42 restated against the oracle."""
    d = json.loads(path.read_text())
    blob = base64.b64decode(d["payload_b64"])
    hdr, samples = O.decode_payload(blob, expect_size=len(blob))
    assert (hdr.codec, hdr.bits) == (d["codec"], d["bits"])
    assert (hdr.width, hdr.height, hdr.count) == (d["width"], d["height"], d["count"])
    for plane, exp in zip(samples, d["expected_samples"]):
        assert plane.ravel().tolist() == exp
    if "expected_values" in d:
        for plane, exp in zip(samples, d["expected_values"]):
            vals = O.dequantize_codes(plane.ravel(), d["bits"], d["range_min"], d["range_max"])
            assert vals.tolist() == exp  # bit-exact float64


@pytest.mark.parametrize("name", scene_names())
def test_container_decode_bit_exact(name):
    """read_layers at every prefix k: every frame's fp64 SoA hashes equal."""
    sc = doc()["scenes"][name]
    data = container(name)
    for k in range(1, sc["layer_count"] + 1):
        info, groups = O.read_layers(data, k)
        assert [(g.start_frame, g.frame_count) for g in groups] == \
            [(g["start"], g["frames"]) for g in sc["groups"]]
        got = [set_sha(O.frame_of(groups, t)) for t in range(sum(g.frame_count for g in groups))]
        assert got == sc["decode"][str(k)], (name, k)
    f0 = renders(f"{name}_frame0")
    _, groups = O.read_layers(data, sc["layer_count"])
    g = O.frame_of(groups, 0)
    for nm in ("positions", "rotations", "scales", "opacities", "sh"):
        assert np.array_equal(getattr(g, nm), f0[nm])


@pytest.mark.parametrize("name", scene_names())
def test_projection_and_render(name):
    sc = doc()["scenes"][name]
    data = container(name)
    arr = renders(name)
    for key, r in sc["renders"].items():
        _, groups = O.read_layers(data, r["k"])
        g = O.frame_of(groups, r["t"])
        cam = camera(name, r["cam"])
        means, covs, depth, colors, opac, rects, idx = O.project_set(g, cam)
        assert np.array_equal(idx, arr[f"{key}_idx"]), key
        assert np.array_equal(rects, arr[f"{key}_rects"]), key
        assert np.array_equal(depth, arr[f"{key}_depth"]), key
        assert np.array_equal(means, arr[f"{key}_means"]), key
        assert np.array_equal(covs, arr[f"{key}_cov"]), key
        assert np.array_equal(colors, arr[f"{key}_colors"]), key
        assert np.array_equal(O.depth_order(depth), arr[f"{key}_order"]), key
        img = O.composite(means, covs, depth, colors, opac, rects, cam)
        assert np.max(np.abs(img - arr[f"{key}_img"])) <= 1e-12, key


def test_group_assignment():
    sc = doc()["scenes"]["deg0_rc"]
    info = O.read_structure(container("deg0_rc"))
    starts = [g["start"] for g in sc["groups"]]
    total = sum(g["frames"] for g in sc["groups"])
    for t in range(total):
        gi = O.group_of(info, t)
        assert starts[gi] <= t
        assert gi == len(starts) - 1 or t < starts[gi + 1]


def test_error_paths_match_reference():
    errs = doc()["errors"]
    blob = container(errs["container"])
    classes = {"CodecError": O.CodecError, "FormatError": O.FormatError,
               "InvalidInputError": O.InvalidInputError}
    for case in errs["cases"]:
        data = bytearray(blob)
        if case["kind"] == "flip":
            data[case["offset"]] ^= 1 << case["bit"]
        elif case["kind"] == "truncate":
            data = data[:case["length"]]
        if case["error"] is None:  # flip in bytes the range decoder never consumes
            O.read_layers(bytes(data), case["k"])
            continue
        with pytest.raises(classes[case["error"]]) as ei:
            O.read_layers(bytes(data), case["k"])
        assert str(ei.value) == case["message"], case


def test_progressive_reconstruct_and_render():
    layers, deltas, cam, d, a = progressive_inputs()
    for key, c in d["cases"].items():
        g = O.reconstruct_frame(layers, deltas, c["t"], c["k"])
        for nm in ("positions", "rotations", "scales", "opacities", "sh"):
            assert np.array_equal(getattr(g, nm), a[f"recon_{key}_{nm}"]), (key, nm)
        img = O.render_progressive(layers, c["k"], deltas, c["t"], cam)
        assert np.max(np.abs(img - a[f"img_{key}"])) <= 1e-12, key


def test_progressive_range_errors():
    layers, deltas, cam, d, a = progressive_inputs()
    with pytest.raises(O.InvalidInputError, match="layer 4 out of range 1..3"):
        O.render_progressive(layers, 4, deltas, 0, cam)
    with pytest.raises(O.InvalidInputError, match=r"frame index 9 out of range 0..4"):
        O.reconstruct_frame(layers, deltas, 9, 1)


def test_tile_keys_consistent_with_counts():
    arr = renders("c1mini_rc")
    rects = arr["k2_t0_axis_rects"][arr["k2_t0_axis_order"]]
    counts = O.tile_counts(rects)
    tiles, ranks = O.tile_keys(rects, 96)
    assert tiles.size == counts.sum()
    assert np.all(np.diff(tiles) >= 0)
    for t in np.unique(tiles)[:20]:
        assert np.all(np.diff(ranks[tiles == t]) > 0)


def test_render2d_and_psnr_oracle():
    """render(list[Splat2D]) (render.py:359-379) and psnr (metrics.py:31-38)
    restated in the oracle, pinned to the reference's outputs."""
    from golden_util import Cam, doc, renders
    d = doc()["render2d"]
    r = renders("render2d")
    cam = Cam.from_json(d["camera"])
    img = O.render2d(r["means"], r["cov"], r["depth"], r["colors"], r["opac"], cam)
    assert np.max(np.abs(img - r["img"])) <= 1e-12
    assert O.psnr(r["img"], r["img_half"]) == d["psnr_full_half"]
    assert O.psnr(r["img"], r["img"]) == d["psnr_same"] == 99.0
    empty = O.render2d(np.zeros((0, 2)), np.zeros((0, 2, 2)), [], np.zeros((0, 3)), [], cam)
    assert np.array_equal(empty, np.tile(np.asarray(cam.background), (cam.height, cam.width, 1)))


def test_ssim_oracle():
    """ssim (metrics.py:40-65) restated separably, pinned to the reference."""
    from golden_util import doc, renders
    d = doc()["render2d"]
    r = renders("render2d")
    assert abs(O.ssim(r["img"], r["img_half"]) - d["ssim_full_half"]) <= 1e-12
    assert abs(O.ssim(r["img"], r["img"]) - d["ssim_same"]) <= 1e-12
