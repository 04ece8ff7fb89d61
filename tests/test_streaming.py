"""Segment-fed progressive decode (paper_2509_17513_b200/streaming.py):
the manifest and segments are pinned to the reference's stream fixture
(pkg/conformance/stream/{manifest,expected}.json, copied into
tests/golden/conformance/stream/); segment containers decode bit-exactly
like the whole container (CPU oracle); the GPU player renders every prefix
exactly like the whole-container path."""

from __future__ import annotations

import json

import numpy as np
import pytest

from golden_util import GOLDEN, camera, container
from oracle import oracle as O
from paper_2509_17513_b200 import streaming as S
from paper_2509_17513_b200.errors import InvalidInputError, StreamError

STREAM = GOLDEN / "conformance" / "stream"


def _scene():
    data = container("stream60")
    return data, S.emit_manifest(data)


def test_manifest_matches_reference_fixture():
    data, m = _scene()
    ref = (STREAM / "manifest.json").read_bytes().strip()
    assert m.to_json_bytes() == ref
    assert S.Manifest.from_json_bytes(ref) == m
    assert m.frame_count == 4
    assert m.cum_bytes_per_frame(6) == sum(g.cum_bytes[5] for g in m.groups) / 4
    assert m.cum_bytes_per_frame(1, group=1) == m.groups[1].cum_bytes[0] / m.groups[1].frames
    with pytest.raises(InvalidInputError):
        m.cum_bytes_per_frame(7)


def test_segments_are_the_directory_ranges():
    data, m = _scene()
    info = O.read_structure(data)
    for gi, g in enumerate(m.groups):
        for l in range(1, m.layers + 1):
            seg = S.segment(data, gi, l)
            assert len(seg) == g.layer_bytes[l - 1]
            assert len(S.parse_payload_stream(seg)) == len(info.groups[gi].channels[l - 1])


def test_segment_containers_decode_like_the_container():
    data, m = _scene()
    for gi, g in enumerate(m.groups):
        segs = {}
        for l in range(1, m.layers + 1):
            segs[l] = S.segment(data, gi, l)
            c = S.segment_container(m, gi, segs)
            _, full = O.read_layers(data, l)
            _, part = O.read_layers(c, l)
            for t in range(g.frames):
                a, b = O.frame_of(full, g.start + t), O.frame_of(part, t)
                for nm in ("positions", "rotations", "scales", "opacities", "sh"):
                    assert np.array_equal(getattr(a, nm), getattr(b, nm)), (gi, l, t, nm)


def test_expected_frame0_values():
    data, m = _scene()
    exp = json.loads((STREAM / "expected.json").read_text())
    c = S.segment_container(m, 0, {l: S.segment(data, 0, l) for l in range(1, m.layers + 1)})
    _, gs = O.read_layers(c, m.layers)
    f0 = O.frame_of(gs, 0)
    assert np.array_equal(f0.positions.ravel(), np.asarray(exp["frame0_positions"]))
    assert np.array_equal(f0.opacities, np.asarray(exp["frame0_opacities"]))
    assert np.array_equal(f0.rotations.ravel()[:len(exp["frame0_rotations_head"])],
                          np.asarray(exp["frame0_rotations_head"]))
    assert np.array_equal(f0.sh.ravel()[:len(exp["frame0_sh_head"])], np.asarray(exp["frame0_sh_head"]))
    assert list(m.groups[0].gauss_counts) == exp["layer_counts"]


def test_segment_errors():
    data, m = _scene()
    seg = S.segment(data, 0, 1)
    first = S.parse_payload_stream(seg)[0][1]
    with pytest.raises(StreamError):
        S.segment_container(m, 0, {1: seg[len(first):]})
    with pytest.raises(InvalidInputError):
        S.segment_container(m, 0, {2: seg})
    with pytest.raises(InvalidInputError):
        S.segment(data, 0, 7)


@pytest.mark.gpu
def test_progressive_player_gpu():
    """Layers arrive one at a time (group 1 before group 0); after each
    arrival every frame renders bit-identically to decoding the whole
    container at that prefix, and decodes to the oracle's values."""
    import paper_2509_17513_b200 as gsvb
    data, m = _scene()
    cam = camera("stream60", "oblique")
    player = S.SegmentVideo(m)
    try:
        with pytest.raises(StreamError):
            player.render(0, cam)
        for l in range(1, m.layers + 1):
            for gi in (1, 0):
                player.add_segment(gi, l, S.segment(data, gi, l))
            _, groups = O.read_layers(data, l)
            with gsvb.DeviceVideo(data, l) as whole:
                for t in range(m.frame_count):
                    a = player.render(t, cam).cpu().numpy()
                    b = whole.render(t, cam).cpu().numpy()
                    assert np.array_equal(a, b), (l, t)
                    got = player.frame(t)
                    ref = O.frame_of(groups, t)
                    for nm in ("positions", "rotations", "scales", "opacities", "sh"):
                        assert np.array_equal(getattr(got, nm), getattr(ref, nm)), (l, t, nm)
    finally:
        player.close()


@pytest.mark.gpu
def test_decode_segment_gpu():
    """_decode_segment semantics: valid segments decode; a missing payload is
    a StreamError; a corrupted payload raises the reference's CodecError."""
    from paper_2509_17513_b200.errors import CodecError
    data, m = _scene()
    for gi in range(len(m.groups)):
        for l in range(1, m.layers + 1):
            S.decode_segment(S.segment(data, gi, l), m, gi, l)
    seg = S.segment(data, 0, 2)
    pl = S.parse_payload_stream(seg)
    with pytest.raises(StreamError, match="expected"):
        S.decode_segment(b"".join(raw for _, raw in pl[:-1]), m, 0, 2)
    bad = bytearray(seg)
    n0 = len(pl[0][1])
    bad[n0 - 1] ^= 0xFF  # the first payload's CRC
    with pytest.raises(CodecError) as e:
        S.decode_segment(bytes(bad), m, 0, 2)
    with pytest.raises(Exception) as e_ref:  # the oracle's own CodecError class
        O.decode_payload(pl[0][1][:-1] + bytes([pl[0][1][-1] ^ 0xFF]))
    assert str(e.value) == str(e_ref.value)
