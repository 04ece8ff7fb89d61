"""GPU encoder: quantisation + codec-1 range coding on
the device, byte-identical to the reference encoder.

* whole containers against the reference-written fixtures
  (tests/golden/containers/*.gsv, encode_sequence of gen_synthetic_scene);
* gsv_encode_runs against the host restatement gsv_encode_reference_body
  (codec.py:137-163) on runs built to hit every branch: constant / smooth /
  ramp / random planes (RAW planes, whole-run raw fallback), 8/16/32-bit,
  odd geometries;
* error behaviour of the quantiser (non-finite input).
"""

import ctypes
import struct
import zlib

import numpy as np
import pytest

from golden_util import container, doc, scene_names
from test_tooling import _spec

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sess():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2509_17513_b200.api import Session
    return Session()


@pytest.mark.parametrize("name", scene_names())
def test_gpu_encoder_reproduces_reference_bytes(sess, name):
    from paper_2509_17513_b200.encode import EncodeConfig, encode_stream
    from paper_2509_17513_b200.synth import iter_frames
    rec = doc()["scenes"][name]["recipe"]
    spec = _spec(rec)
    c = rec["cfg"]
    cfg = EncodeConfig(layer_count=c["layer_count"], prune_fraction=0.0, motion_threshold=0.0025,
                       codec=c["codec"], fixed_group_length=c.get("fixed_group_length"))
    out = encode_stream(lambda: iter_frames(spec, rec["seed"]), cfg, codecs=(0, 1), device=sess)
    assert out[c["codec"]] == container(name)
    host = encode_stream(lambda: iter_frames(spec, rec["seed"]), cfg, codecs=(0, 1), threads=4)
    assert out == host


def _runs():
    rng = np.random.default_rng(7)
    out = []
    for bits in (8, 16, 32):
        top = (1 << bits) - 1
        mask = np.uint64(top)
        for (count, h, w) in ((1, 1, 1), (3, 5, 7), (4, 17, 16), (6, 31, 33)):
            n = count * h * w
            base = rng.integers(0, top + 1, size=(h, w), dtype=np.uint64)
            smooth = (base[None] + np.arange(count, dtype=np.uint64)[:, None, None] * np.uint64(3)) & mask
            out.append(("smooth", bits, smooth.astype(np.uint32)))
            out.append(("random", bits, rng.integers(0, top + 1, size=(count, h, w), dtype=np.uint64)
                        .astype(np.uint32)))
            out.append(("constant", bits, np.full((count, h, w), top // 3, np.uint32)))
            ramp = (np.arange(n, dtype=np.uint64).reshape(count, h, w) * np.uint64(1000)) & mask
            out.append(("ramp", bits, ramp.astype(np.uint32)))
            # mostly smooth with one noisy plane (RAW plane inside a coded run)
            mix = smooth.copy()
            mix[count // 2] = rng.integers(0, top + 1, size=(h, w), dtype=np.uint64).astype(np.uint32)
            out.append(("mixed", bits, mix))
    return out


def test_gpu_range_coder_matches_host_restatement(sess):
    import torch

    from paper_2509_17513_b200 import _lib
    L = _lib.load()
    runs = _runs()
    dev = torch.device("cuda", sess.device)
    le = {8: np.uint8, 16: np.dtype("<u2"), 32: np.dtype("<u4")}
    samples = [torch.from_numpy(np.ascontiguousarray(a.astype(le[b])).view(np.uint8).reshape(-1).copy()).to(dev)
               for _, b, a in runs]
    caps = [int(L.gsv_encode_body_capacity(a.shape[0], a.shape[2], a.shape[1], b)) for _, b, a in runs]
    bodies = [torch.zeros(c, dtype=torch.uint8, device=dev) for c in caps]
    arr = (_lib.EncodeRun_t * len(runs))()
    for i, (_, b, a) in enumerate(runs):
        arr[i] = _lib.EncodeRun_t(samples[i].data_ptr(), bodies[i].data_ptr(), a.shape[0], a.shape[2],
                                  a.shape[1], b, 0, 0, 0)
    torch.cuda.synchronize()
    _lib.check(L.gsv_encode_runs(sess.handle, arr, len(runs)))
    kinds = set()
    for i, (kind, b, a) in enumerate(runs):
        count, h, w = a.shape
        flat = np.ascontiguousarray(a, dtype=np.uint32)
        cap = flat.size * (b // 8) + 1 + count + 64
        ref = np.empty(cap, np.uint8)
        n = L.gsv_encode_reference_body(flat.ctypes.data, count, h, w, b, ref.ctypes.data, cap)
        assert n > 0
        got = bodies[i][:int(arr[i].body_len)].cpu().numpy()
        assert got.tobytes() == ref[:n].tobytes(), (kind, b, a.shape)
        raw = np.ascontiguousarray(a.astype(le[b])).tobytes()
        assert int(arr[i].checksum) == zlib.crc32(raw) & 0xFFFFFFFF
        kinds.add(("whole_raw" if ref[0] == 1 else
                   ("raw_plane" if 1 in ref[1:1 + count] else "coded")))
    assert kinds == {"whole_raw", "raw_plane", "coded"}


def test_gpu_quantizer_rejects_non_finite(sess):
    import torch

    from paper_2509_17513_b200 import _lib
    from paper_2509_17513_b200.errors import InvalidInputError
    L = _lib.load()
    v = torch.zeros((2, 10), dtype=torch.float64, device="cuda")
    v[1, 3] = float("nan")
    planes = torch.empty(2 * 16, dtype=torch.uint8, device="cuda")
    qc = (_lib.QuantChannel_t * 1)()
    qc[0] = _lib.QuantChannel_t(v.data_ptr(), planes.data_ptr(), 10, 2, 10, 4, 3, 8, 0.0, 0.0)
    torch.cuda.synchronize()
    with pytest.raises(InvalidInputError, match="non-finite"):
        _lib.check(L.gsv_quantize_channels(sess.handle, qc, 1))


def test_gpu_quantizer_matches_numpy(sess):
    """quantize_channel semantics incl. the degenerate range and padding."""
    import torch

    from paper_2509_17513_b200 import _lib
    from paper_2509_17513_b200.encode import _planes, _quantize
    L = _lib.load()
    rng = np.random.default_rng(3)
    cases = [(rng.normal(size=(3, 50)) * 1e-3 + 0.25, 8), (rng.uniform(-7, 9, size=(4, 37)), 16),
             (np.full((2, 5), 0.1), 8), (rng.uniform(-1e6, 1e6, size=(2, 30)), 32),
             (np.array([[1.0, 1.0 + 2 ** -40]]), 16)]
    for vals, bits in cases:
        f, n = vals.shape
        codes, rmin, rmax = _quantize(vals.ravel(), bits)
        want = _planes(codes.reshape(vals.shape))
        h, w = want.shape[1], want.shape[2]
        dv = torch.from_numpy(vals).to("cuda")
        planes = torch.zeros(f * h * w * (bits // 8), dtype=torch.uint8, device="cuda")
        qc = (_lib.QuantChannel_t * 1)()
        qc[0] = _lib.QuantChannel_t(dv.data_ptr(), planes.data_ptr(), n, f, n, w, h, bits, 0.0, 0.0)
        torch.cuda.synchronize()
        _lib.check(L.gsv_quantize_channels(sess.handle, qc, 1))
        assert (float(qc[0].range_min), float(qc[0].range_max)) == (rmin, rmax)
        got = planes.cpu().numpy().view(want.dtype).reshape(want.shape)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("case", ["prune_fractions", "fixed_groups_deg3", "deg0_wide", "large_motion"])
def test_gpu_encoder_matches_host_encoder(sess, case):
    """Encoder options the fixtures do not pin (pruning, custom layer
    fractions, fixed group lengths, SH degrees 0 and 3, 32-bit positions,
    strong motion that cuts many groups): GPU bytes == host bytes, both
    codecs."""
    from paper_2509_17513_b200.encode import EncodeConfig, encode_stream
    from paper_2509_17513_b200.synth import SceneSpec, iter_frames
    if case == "prune_fractions":
        spec = SceneSpec(count=5000, frames=6, sh_degree=1, amplitude=0.002, rotation_amplitude=0.02,
                         scale_amplitude=0.001, opacity_amplitude=0.01, sh_amplitude=0.01)
        cfg = EncodeConfig(layer_count=3, layer_fractions=(0.2, 0.3, 0.5), prune_fraction=0.4)
    elif case == "fixed_groups_deg3":
        spec = SceneSpec(count=3000, frames=7, sh_degree=3, amplitude=0.001, rotation_amplitude=0.05,
                         scale_amplitude=0.001, opacity_amplitude=0.02, sh_amplitude=0.02)
        cfg = EncodeConfig(layer_count=4, prune_fraction=0.1, fixed_group_length=3)
    elif case == "deg0_wide":
        spec = SceneSpec(count=2000, frames=4, sh_degree=0, amplitude=0.5, position_extent=80.0)
        cfg = EncodeConfig(layer_count=2, prune_fraction=0.0)
    else:
        spec = SceneSpec(count=4000, frames=8, sh_degree=1, amplitude=0.02, rotation_amplitude=0.3,
                         scale_amplitude=0.01, opacity_amplitude=0.1, sh_amplitude=0.1)
        cfg = EncodeConfig(layer_count=6, prune_fraction=0.0)
    host = encode_stream(lambda: iter_frames(spec, 11), cfg, codecs=(0, 1), threads=4)
    gpu = encode_stream(lambda: iter_frames(spec, 11), cfg, codecs=(0, 1), device=sess)
    assert gpu[0] == host[0]
    assert gpu[1] == host[1]
