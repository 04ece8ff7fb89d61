"""GPU parity at BASELINE scale, through the production path.

The renders the bench times project straight from the decoded code planes
(PlaneLoader: codes dequantised in registers), so these tests check that path
(`DeviceVideo.project_debug`, `DeviceVideo.render`) against the CPU oracle on
BASELINE geometry:

* config 2 (300k Gaussians, 6 layers, 1080p), one 30-frame group -- the
  bench's group length, so every codec-1 run carries 29 range-coded planes
  under one persistent adaptive model -- both codecs, the axis camera (about
  30% of the splats tie exactly in fp64 depth, so the stable index
  tie-break decides the order) and an oblique one: rects, fp64 depth, stable
  depth order and per-splat tile counts bit-exact, images within max-abs
  2e-3, |dPSNR| <= 0.01 dB against the unquantised source render, u8 output
  equal to write_ppm's rounding;
* config 2 codec 1: the decoded integer codes of frames 1, 15 and 29 of the
  30-frame group (model persistence across 29 planes) against the oracle;
* config 5: a 3M-splat 4K frame; and 1M splats at 3840x2160 (32,400 tiles: round-1 binning)
  and at 4096x2304 (36,864 tiles: above the binning limit, emit + sort);
* config 4: two of the 16 ring cameras at 500k splats;
* config 3: 1M splats in 2-frame adaptive groups, both codecs (codes of a
  range-coded group, projection, image, render_sequence's frames);
* depth-order robustness: a near-planar scene and one whose depth range is
  stretched by a far outlier (long runs of equal truncated sort keys).

Bars (BASELINE.json north_star): bit-exact integer symbols, rects, tile counts
and order; max-abs 2e-3 per pixel channel; |dPSNR| <= 0.01 dB.
"""

import numpy as np
import pytest

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


def _encode(cfg, frames, codecs=(0, 1)):
    from paper_2509_17513_b200.encode import EncodeConfig, encode_stream
    from paper_2509_17513_b200.synth import iter_frames
    spec = cfg.spec(frames)
    enc = EncodeConfig(layer_count=cfg.layers, prune_fraction=0.0, motion_threshold=0.0025)
    blobs = encode_stream(lambda: iter_frames(spec, cfg.seed), enc, codecs=codecs, device=True,
                          positions_source=lambda: iter_frames(spec, cfg.seed, positions_only=True))
    return blobs, spec


def _source_frames(spec, seed, wanted):
    from paper_2509_17513_b200.synth import iter_frames
    out = {}
    for t, f in enumerate(iter_frames(spec, seed)):
        if t in wanted:
            out[t] = f
        if len(out) == len(wanted):
            break
    return out


def _oracle_frames(data, k, frames):
    """Oracle decode of group 0 (layers <= k) and the listed frames."""
    info = O.read_structure(data)
    vals = O.decode_group_codes(data, info, 0, k)
    sets = O.assemble(info, info.groups[0], vals, k, only=frames)
    return info, vals, dict(zip(frames, sets))


def _write_ppm_u8(img):
    """write_ppm's quantisation (render.py:165-169)."""
    return np.clip(np.floor(np.asarray(img, np.float64) * 255.0 + 0.5), 0, 255).astype(np.uint8)


def check_projection(v, t, cam, oset):
    """Production projection of frame t vs the oracle's project_set: rects,
    survivors, fp64 depth, stable depth order and tile counts bit-exact."""
    prect, pdepth, porder, ptiles, nvis = v.project_debug(t, cam)
    means, covs, depth, colors, opac, rects, idx = O.project_set(oset, cam)
    assert nvis == idx.size
    assert np.array_equal(prect[idx].astype(np.int64), rects)
    culled = np.ones(prect.shape[0], bool)
    culled[idx] = False
    assert not prect[culled].any()
    assert np.array_equal(pdepth[idx], depth)
    assert np.array_equal(porder[:nvis], idx[O.depth_order(depth)])
    assert np.array_equal(ptiles[idx], O.tile_counts(rects))
    return means, covs, depth, colors, opac, rects


def check_image(v, t, cam, proj, gt=None):
    """Production render of frame t vs the oracle composite (max-abs), the
    u8 output vs write_ppm, and dPSNR against a ground-truth render."""
    import torch
    img32 = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device="cuda")
    u8 = torch.empty((cam.height, cam.width, 3), dtype=torch.uint8, device="cuda")
    _, st = v.render(t, cam, out=img32, out_u8=u8, stats=True)
    img = img32.cpu().numpy().astype(np.float64)
    ref = O.composite(*proj, cam)
    err = float(np.max(np.abs(img - ref)))
    assert err <= MAX_ABS, err
    assert st["n_visible"] == proj[5].shape[0]
    assert st["n_keys"] == int(O.tile_counts(proj[5]).sum())
    got8 = u8.cpu().numpy()
    assert np.array_equal(got8, _write_ppm_u8(img))  # write_ppm of the returned image, exactly
    d8 = np.abs(got8.astype(np.int16) - _write_ppm_u8(ref).astype(np.int16))
    assert int(d8.max()) <= 1 and float(np.mean(d8 != 0)) < 1e-3  # vs the oracle's fp64 image
    if gt is not None:
        assert abs(O.psnr(gt, img) - O.psnr(gt, ref)) <= MAX_DPSNR
    return img, ref


# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c2_group(gsvb):
    from paper_2509_17513_b200.configs import CONFIGS
    cfg = CONFIGS["c2"]
    blobs, spec = _encode(cfg, 30)
    return cfg, blobs, spec


def test_c2_codec1_codes_across_29_planes(gsvb, c2_group):
    """Codec 1 with the bench's 30-frame group: runs of 29 or 30 range-coded
    planes (a RAW keyframe plane when coding it does not pay) under one
    adaptive model; the integer
    codes of frames 1, 15 and 29 (all 6 layers, all 23 channels) equal the
    oracle's decode (_rc.py:121-155, 282-301)."""
    cfg, blobs, _ = c2_group
    data = blobs[1]
    info, vals, _ = _oracle_frames(data, cfg.layers, [])
    order = [("position", c) for c in range(3)] + [("rotation", c) for c in range(4)] + \
        [("scales", c) for c in range(3)] + [("opacity", 0)] + \
        [("sh", c) for c in range(3 * (info.sh_degree + 1) ** 2)]
    rc_planes = []
    with gsvb.DeviceVideo(data, cfg.layers) as v:
        assert v.frame_count == 30 and v.group_of(29) == 0
        for t in (1, 15, 29):
            got = v.frame_codes(t).cpu().numpy().astype(np.uint32)
            exp = np.concatenate([np.stack([vals[l][key][0][t] for key in order], axis=1)
                                  for l in range(cfg.layers)])
            assert np.array_equal(got, exp), t
    # the container really carries range-coded runs of 29 planes
    for g in info.groups:
        for l in range(cfg.layers):
            for e in g.channels[l]:
                blob = data[e.offset:e.offset + e.size]
                if blob[0] == 1 and blob[14] == 0:  # codec 1, per-plane mode table
                    modes = blob[15:15 + 30]
                    rc_planes.append(sum(1 for m in modes if m == 0))
    assert min(rc_planes) >= 29 and 29 in rc_planes and 30 in rc_planes


@pytest.mark.parametrize("codec", [0, 1])
@pytest.mark.parametrize("view", ["axis", "oblique"])
def test_c2_projection_order_and_image(gsvb, c2_group, codec, view):
    """Config 2 geometry through the production path: frames 0 and 29 at
    k = 6 and frame 15 at k = 1, projection bit-exact, image / u8 / dPSNR."""
    from paper_2509_17513_b200.configs import axis_camera, oblique_camera
    cfg, blobs, spec = c2_group
    cam = (axis_camera if view == "axis" else oblique_camera)(cfg.width, cfg.height)
    data = blobs[codec]
    src = _source_frames(spec, cfg.seed, {0, 29})
    for k, frames in ((6, (0, 29)), (1, (15,))):
        _, _, osets = _oracle_frames(data, k, list(frames))
        with gsvb.DeviceVideo(data, k) as v:
            for t in frames:
                proj = check_projection(v, t, cam, osets[t])
                if view == "axis" and k == 6:
                    ties = int(np.sum(np.diff(np.sort(proj[2])) == 0))
                    assert ties > 10_000, ties  # the stable tie-break is really exercised
                gt = O.render_set(src[t], cam) if (k == 6 and t in src) else None
                check_image(v, t, cam, proj, gt)


def test_c4_ring_cameras(gsvb):
    """Config 4: 500k splats, two of the 16 ring cameras (views 3 and 10),
    one frame, projection bit-exact and image within tolerance."""
    from paper_2509_17513_b200.configs import CONFIGS
    cfg = CONFIGS["c4"]
    blobs, _ = _encode(cfg, 1, codecs=(0,))
    data = blobs[0]
    cams = cfg.cameras()
    assert len(cams) == 16
    _, _, osets = _oracle_frames(data, cfg.layers, [0])
    with gsvb.DeviceVideo(data, cfg.layers) as v:
        assert v.splat_count(0) == 500_000
        for view in (3, 10):
            proj = check_projection(v, 0, cams[view], osets[0])
            check_image(v, 0, cams[view], proj)


def test_c3_short_groups_1m(gsvb):
    """Config 3 shape: 1M Gaussians, 6 layers, a burst every 2 frames (the
    2-frame adaptive groups), 6 frames = 3 groups, both codecs.  The codes of
    every frame of group 1 (its range-coded second plane under the model the
    keyframe plane trained) equal the oracle's; frame 3 projects bit-exactly
    and renders within tolerance; render_sequence's u8 frames equal the
    per-frame renders for both codecs."""
    import torch
    from paper_2509_17513_b200.configs import CONFIGS
    cfg = CONFIGS["c3"]
    blobs, _ = _encode(cfg, 6)
    info = gsvb.read_structure(blobs[1])
    assert len(info.groups) >= 3 and info.groups[1].start_frame == 2 and info.groups[1].frame_count == 2
    for codec in (0, 1):
        data = blobs[codec]
        info_o = O.read_structure(data)
        vals = O.decode_group_codes(data, info_o, 1, cfg.layers)
        order = [("position", c) for c in range(3)] + [("rotation", c) for c in range(4)] + \
            [("scales", c) for c in range(3)] + [("opacity", 0)] + \
            [("sh", c) for c in range(3 * (info_o.sh_degree + 1) ** 2)]
        with gsvb.DeviceVideo(data, cfg.layers) as v:
            assert v.splat_count(2) == 1_000_000
            for t in (2, 3):  # group 1
                got = v.frame_codes(t).cpu().numpy().astype(np.uint32)
                exp = np.concatenate([np.stack([vals[l][key][0][t - 2] for key in order], axis=1)
                                      for l in range(cfg.layers)])
                assert np.array_equal(got, exp), (codec, t)
            sets = O.assemble(info_o, info_o.groups[1], vals, cfg.layers, only=[1])
            cam = cfg.cameras()[0]
            proj = check_projection(v, 3, cam, sets[0])
            check_image(v, 3, cam, proj)
        import dataclasses
        small = dataclasses.replace(cam, fx=cam.fx / 4, fy=cam.fy / 4, cx=cam.cx / 4, cy=cam.cy / 4,
                                    width=cam.width // 4, height=cam.height // 4)
        seq = gsvb.render_sequence(data, small)
        with gsvb.DeviceVideo(data, cfg.layers) as v:
            for t in range(6):
                u8 = torch.empty((small.height, small.width, 3), dtype=torch.uint8, device="cuda")
                v.render(t, small, out_u8=u8)
                assert torch.equal(seq[t], u8.cpu()), (codec, t)


def test_c5_full_scale_frame(gsvb):
    """Config 5 at its own scale: 3M Gaussians (config 5's recipe), 6 layers,
    one frame at 3840x2160 -- projection, stable order and tile counts
    bit-exact against the oracle, image within 2e-3, u8 = write_ppm."""
    from paper_2509_17513_b200.configs import CONFIGS
    cfg = CONFIGS["c5"]
    blobs, _ = _encode(cfg, 1, codecs=(0,))
    data = blobs[0]
    cam = cfg.cameras()[0]
    _, _, osets = _oracle_frames(data, cfg.layers, [0])
    with gsvb.DeviceVideo(data, cfg.layers) as v:
        assert v.splat_count(0) == 3_000_000
        proj = check_projection(v, 0, cam, osets[0])
        check_image(v, 0, cam, proj)


@pytest.mark.parametrize("size", [(3840, 2160), (4096, 2304)], ids=["4k_binned", "above_32768_tiles"])
def test_c5_geometry_4k(gsvb, size):
    """Config 5 geometry: 1M splats (config 5's scale recipe) at 4K (32,400
    tiles, the round-1 counting placement) and at 4096x2304 (36,864 tiles,
    above the binning limit: emit + tile sort): projection and tile counts
    bit-exact, image within 2e-3 of the oracle."""
    from paper_2509_17513_b200.configs import Config, axis_camera
    cfg = Config("c5geo", 1_000_000, 6, 1, 30, size[0], size[1], 1005)
    blobs, _ = _encode(cfg, 1, codecs=(0,))
    data = blobs[0]
    cam = axis_camera(*size)
    _, _, osets = _oracle_frames(data, cfg.layers, [0])
    with gsvb.DeviceVideo(data, cfg.layers) as v:
        proj = check_projection(v, 0, cam, osets[0])
        ntx, nty = -(-size[0] // 16), -(-size[1] // 16)
        assert (ntx * nty > 32768) == (size[0] == 4096)
        check_image(v, 0, cam, proj)


# ---------------------------------------------------------------------------
def _scene(n, seed, kind):
    from paper_2509_17513_b200.types import GaussianSet
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-0.5, 0.5, size=(n, 3))
    # every splat within 1e-9 of the plane z = 0.1 (depth 2.6 on the axis camera)
    pos[:, 2] = 0.1 + rng.uniform(-1e-9, 1e-9, size=n)
    if kind == "cluster_far":  # one splat 0.4 behind: one truncated key for the whole cluster
        pos[0, 2] = 0.5
    elif kind == "cluster_near":  # one splat 1e-4 behind: runs of a few hundred
        pos[0, 2] = 0.1 + 1e-4
    rot = rng.normal(size=(n, 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    scl = rng.uniform(0.002, 0.01, size=(n, 3))
    opa = rng.uniform(0.2, 1.0, size=n)
    sh = rng.uniform(-0.5, 0.5, size=(n, 12))
    return GaussianSet(pos, rot, scl, opa, sh, 1)


@pytest.mark.parametrize("kind", ["planar", "cluster_near", "cluster_far"])
def test_depth_order_long_tie_runs(gsvb, kind):
    """100k splats with distinct fp64 depths inside 2e-9 (a near-planar
    cluster).  Alone, the 24-bit sort key resolves them exactly; with one
    splat 1e-4 or 0.4 behind, the key's range grows so that runs of a few
    hundred splats (CTA bitonic path), or the whole cluster (CTA merge path),
    share one truncated key.  The exact stable fp64 order (render.py:343) must
    come back in every case, and the image must match the oracle."""
    from paper_2509_17513_b200.configs import axis_camera
    g = _scene(100_000, 5, kind)
    cam = axis_camera(640, 480)
    prect, pdepth, porder, ptiles, nvis = gsvb.project_debug(g, cam)
    means, covs, depth, colors, opac, rects, idx = O.project_set(g, cam)
    assert nvis == idx.size
    assert np.unique(depth).size > 50_000  # mostly distinct depths
    assert np.array_equal(pdepth[idx], depth)
    assert np.array_equal(porder[:nvis], idx[O.depth_order(depth)])
    img = gsvb.render_set(g, cam).pixels
    ref = O.composite(means, covs, depth, colors, opac, rects, cam)
    assert np.max(np.abs(img - ref)) <= MAX_ABS
