"""render_sequence (gsv_render_sequence_host): the reference's decode_video
+ render_set + write_ppm of every frame (pipeline.py:350-359,
render.py:382-385, 165-169) as one pipelined call.  Its u8 frames must equal
the per-frame path's (DeviceVideo.render with the u8 output) bit for bit,
for raw containers (the per-group upload/open/render pipeline) and
range-coded ones (one open of every group), for every prefix, for group
lists, and a corrupt payload must raise the error decode_video raises."""

import numpy as np
import pytest
import torch

from golden_util import camera, container, scene_names

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gsvb():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2509_17513_b200 as m
    return m


def _per_frame(gsvb, data, k, cam, groups=None):
    info = gsvb.read_structure(data)
    gl = list(range(len(info.groups))) if groups is None else list(groups)
    out = []
    with gsvb.DeviceVideo(data, k, group_list=gl) as v:
        for t in range(v.frame_count):
            u8 = torch.empty((cam.height, cam.width, 3), dtype=torch.uint8, device="cuda")
            v.render(t, cam, out_u8=u8)
            out.append(u8.cpu())
    return torch.stack(out)


@pytest.mark.parametrize("name", scene_names())
def test_sequence_matches_per_frame_render(gsvb, name):
    data = container(name)
    cam = camera(name, "oblique")
    L = gsvb.read_structure(data).layer_count
    for k in sorted({1, L}):
        got = gsvb.render_sequence(data, cam, up_to_layer=k)
        ref = _per_frame(gsvb, data, k, cam)
        assert got.shape == ref.shape
        assert torch.equal(got, ref), (name, k)


@pytest.mark.parametrize("ring", ["0", "1"])
def test_sequence_group_list_and_pinned_source(gsvb, ring, monkeypatch):
    """Groups in any order, from a pinned host tensor; every group in its own
    device slot, or (GSV_SEQ_RING=1) the ring of 3 slots reused as groups
    finish."""
    monkeypatch.setenv("GSV_SEQ_RING", ring)
    import bench
    from paper_2509_17513_b200.encode import EncodeConfig, encode_stream
    from paper_2509_17513_b200.synth import benchmark_spec, iter_frames
    spec = benchmark_spec(20_000, 15, 3)  # 5 raw groups: the ring wraps
    blobs = encode_stream(lambda: iter_frames(spec, 7), EncodeConfig(layer_count=3, prune_fraction=0.0),
                          codecs=(0, 1))
    cam = bench.camera(type("A", (), {"width": 320, "height": 240})())
    for codec in (0, 1):
        data = blobs[codec]
        host = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
        for gl in ([0, 1, 2, 3, 4], [2, 0, 4, 3]):
            got = gsvb.render_sequence(host, cam, up_to_layer=2, groups=gl)
            ref = _per_frame(gsvb, data, 2, cam, gl)
            assert torch.equal(got, ref), (codec, gl)


def test_sequence_corrupt_payload_raises_like_decode_video(gsvb):
    from paper_2509_17513_b200.errors import CodecError
    data = bytearray(container("s1_raw"))
    info = gsvb.read_structure(bytes(data))
    e = info.groups[-1].channels[0][0]  # last group: the pipeline has rendered earlier groups
    data[e.offset + e.size // 2] ^= 0x5A
    cam = camera("s1_raw", "axis")
    with pytest.raises(CodecError) as a:
        gsvb.decode_video(bytes(data))
    with pytest.raises(CodecError) as b:
        gsvb.render_sequence(bytes(data), cam)
    assert str(a.value) == str(b.value)


def test_sequence_resident_device_outputs(gsvb):
    """The container already in HBM (no uploads), device u8 and fp32 outputs:
    the path the bench's resident step runs."""
    import bench
    from paper_2509_17513_b200.encode import EncodeConfig, encode_stream
    from paper_2509_17513_b200.synth import benchmark_spec, iter_frames
    spec = benchmark_spec(20_000, 12, 3)
    blobs = encode_stream(lambda: iter_frames(spec, 11), EncodeConfig(layer_count=3, prune_fraction=0.0),
                          codecs=(0, 1))
    cam = bench.camera(type("A", (), {"width": 256, "height": 192})())
    for codec in (0, 1):
        data = blobs[codec]
        dev = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
        ref = _per_frame(gsvb, data, 3, cam)
        u8 = [torch.empty((192, 256, 3), dtype=torch.uint8, device="cuda") for _ in range(ref.shape[0])]
        f32 = [torch.empty((192, 256, 3), dtype=torch.float32, device="cuda") for _ in range(ref.shape[0])]
        assert gsvb.render_sequence(data, cam, up_to_layer=3, resident=dev, outs=f32, outs_u8=u8) is None
        got = torch.stack([t.cpu() for t in u8])
        assert torch.equal(got, ref), codec
        with gsvb.DeviceVideo(data, 3) as v:
            img = v.render(5, cam)
        assert torch.equal(f32[5], img)


def test_sequence_argument_errors(gsvb):
    from paper_2509_17513_b200.errors import InvalidInputError
    data = container("s1_raw")
    cam = camera("s1_raw", "axis")
    with pytest.raises(InvalidInputError):
        gsvb.render_sequence(data, cam, groups=[0, 7])
    with pytest.raises(InvalidInputError):
        gsvb.render_sequence(data, cam, up_to_layer=9)
    with pytest.raises(InvalidInputError):  # a group listed twice
        gsvb.render_sequence(data, cam, groups=[0, 0])
    with pytest.raises(InvalidInputError):  # wrong output shape
        gsvb.render_sequence(data, cam, out=torch.empty((1, 2, 3, 3), dtype=torch.uint8))


def test_sequence_pieces(gsvb):
    """Frame ranges of groups (a rank's shard when raw groups are split
    between ranks): the frames equal per-frame renders, for both codecs,
    resident and from host bytes; an empty or out-of-range range is an
    InvalidInputError."""
    import bench
    from paper_2509_17513_b200.encode import EncodeConfig, encode_stream
    from paper_2509_17513_b200.errors import InvalidInputError
    from paper_2509_17513_b200.synth import benchmark_spec, iter_frames
    spec = benchmark_spec(20_000, 12, 3)
    blobs = encode_stream(lambda: iter_frames(spec, 13), EncodeConfig(layer_count=2, prune_fraction=0.0),
                          codecs=(0, 1))
    cam = bench.camera(type("A", (), {"width": 256, "height": 192})())
    pieces = [(1, 1, 3), (0, 0, 2), (3, 2, 3)]
    for codec in (0, 1):
        data = blobs[codec]
        info = gsvb.read_structure(data)
        assert all(g.frame_count == 3 for g in info.groups)
        full = _per_frame(gsvb, data, 2, cam)
        want = torch.stack([full[info.groups[g].start_frame + f] for g, f0, f1 in pieces for f in range(f0, f1)])
        got = gsvb.render_sequence(data, cam, up_to_layer=2, pieces=pieces)
        assert torch.equal(got, want), codec
        dev = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
        u8 = [torch.empty((192, 256, 3), dtype=torch.uint8, device="cuda") for _ in range(want.shape[0])]
        gsvb.render_sequence(data, cam, up_to_layer=2, pieces=pieces, resident=dev, outs_u8=u8)
        assert torch.equal(torch.stack([t.cpu() for t in u8]), want), codec
        with pytest.raises(InvalidInputError):
            gsvb.render_sequence(data, cam, pieces=[(0, 2, 2)])
        with pytest.raises(InvalidInputError):
            gsvb.render_sequence(data, cam, pieces=[(0, 0, 4)])


def test_render_batch_output_lists(gsvb):
    """render_batch takes output j for frame j from lists at least as long as
    the frame list (a rank's buffers are sized for its largest shard)."""
    from paper_2509_17513_b200.errors import InvalidInputError
    data = container("s1_raw")
    cam = camera("s1_raw", "axis")
    with gsvb.DeviceVideo(data) as v:
        outs = [torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device="cuda") for _ in range(5)]
        v.render_batch([1, 0], cam, outs=outs)
        assert torch.equal(outs[0], v.render(1, cam)) and torch.equal(outs[1], v.render(0, cam))
        with pytest.raises(InvalidInputError):
            v.render_batch([0, 1, 0], cam, outs=outs[:2])
