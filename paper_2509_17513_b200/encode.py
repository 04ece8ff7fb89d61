"""Container encoder (benchmark input tooling; not on the decode/render path).

Produces `.gsv` bytes identical to the reference encoder encode_sequence
(pipeline.py:137-347 of /root/reference/pkg/src/gsv) for the same frames and
configuration -- checked byte-for-byte in tests/test_tooling.py against
reference-encoded fixtures -- but streams group by group (the reference holds
every frame in fp64, which the large BASELINE configs cannot afford), and
range-codes runs in parallel native threads (libgsv_b200's
gsv_encode_reference_body, a restatement of _rc.encode_bittree /
codec._encode_reference_body).  One quantisation pass can emit the container
under several codecs at once.
"""

from __future__ import annotations

import math
import os
import struct
import sys
import time
import zlib
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Callable, Iterable, Sequence

import numpy as np

from .errors import InvalidInputError
from .types import ATTRIBUTE_CODES, GaussianSet, sh_coeff_count

_LE = {8: "<u1", 16: "<u2", 32: "<u4"}
# container channel order inside a layer = sorted ChannelId (attribute name, component)
_ATTRS_SORTED = ("opacity", "position", "rotation", "scales", "sh")
_WIDTH = {"position": 3, "rotation": 4, "scales": 3, "opacity": 1}


@dataclass(frozen=True)
class EncodeConfig:
    """Subset of pipeline.EncodeConfig (pipeline.py:55-110) that shapes the bitstream."""

    layer_count: int = 6
    layer_fractions: tuple | None = None
    volume_weight: float = 1e5
    motion_threshold: float = 0.0025
    prune_fraction: float = 0.4
    position_bits: int = 16
    wide_extent: float = 50.0
    codec: int = 1
    fps: tuple = (30, 1)
    fixed_group_length: int | None = None

    def fractions(self) -> tuple:
        if self.layer_fractions is not None:
            return tuple(float(f) for f in self.layer_fractions)
        return tuple(1.0 / self.layer_count for _ in range(self.layer_count))


# ---- encoder-side helpers (gaussians.py:204-307, quantize.py:62-167) -------

def _keep_after_prune(opacities: np.ndarray, fraction: float) -> np.ndarray:
    n = opacities.shape[0]
    drop = int(np.floor(fraction * n))
    if drop == 0:
        return np.arange(n, dtype=np.int64)
    removed = np.lexsort((-np.arange(n), opacities))[:drop]
    mask = np.ones(n, dtype=bool)
    mask[removed] = False
    return np.nonzero(mask)[0].astype(np.int64)


def _significance_rank(g: GaussianSet, weight: float) -> np.ndarray:
    vol = (4.0 / 3.0) * np.pi * np.prod(g.scales, axis=1)
    psi = g.opacities + weight * vol
    if not np.all(np.isfinite(psi)):
        raise InvalidInputError("non-finite significance values")
    return np.argsort(-psi, kind="stable")


def _layer_sizes(n: int, fractions: Sequence[float]) -> list:
    sizes, left = [], n
    for f in fractions[:-1]:
        k = min(int(np.floor(f * n + 0.5)), left)
        sizes.append(k)
        left -= k
    sizes.append(left)
    return sizes


def _f32_cover(values: np.ndarray):
    vmin, vmax = float(values.min()), float(values.max())
    if vmax == vmin:
        vmax = vmin + 1e-6
    lo = np.float32(vmin)
    if float(lo) > vmin:
        lo = np.nextafter(lo, np.float32(-np.inf), dtype=np.float32)
    hi = np.float32(vmax)
    if float(hi) < vmax:
        hi = np.nextafter(hi, np.float32(np.inf), dtype=np.float32)
    while float(hi) <= float(lo):
        hi = np.nextafter(hi, np.float32(np.inf), dtype=np.float32)
    return lo, hi


def _quantize(values: np.ndarray, bits: int):
    if not np.all(np.isfinite(values)):
        raise InvalidInputError("non-finite channel values")
    lo32, hi32 = _f32_cover(values)
    lo, hi = float(lo32), float(hi32)
    top = float(2 ** bits - 1)
    codes = np.clip(np.floor((values - lo) / (hi - lo) * top + 0.5), 0, top)
    return codes.astype(_LE[bits]), float(lo32), float(hi32)


def _plane_shape(n: int):
    w = int(np.ceil(np.sqrt(n)))
    return w, int(np.ceil(n / w))


def _planes(codes: np.ndarray):
    """(F, n) codes -> (F, H, W) planes padded with each frame's last code."""
    f, n = codes.shape
    w, h = _plane_shape(n)
    out = np.empty((f, w * h), dtype=codes.dtype)
    out[:, :n] = codes
    out[:, n:] = codes[:, -1:]
    return out.reshape(f, h, w)


def _payload(planes: np.ndarray, bits: int, codec: int, lib) -> bytes:
    count, h, w = planes.shape
    if max(w, h, count) > 0xFFFF:
        raise InvalidInputError("plane run exceeds u16 geometry limits")
    raw = np.ascontiguousarray(planes, dtype=_LE[bits]).tobytes()
    crc = zlib.crc32(raw) & 0xFFFFFFFF
    if codec == 0:
        body = raw
    elif codec == 1:
        samples = np.ascontiguousarray(planes, dtype=np.uint32)
        cap = len(raw) + 1 + count + 64
        out = np.empty(cap, np.uint8)
        n = lib.gsv_encode_reference_body(samples.ctypes.data, count, h, w, bits,
                                          out.ctypes.data, cap)
        if n < 0:
            raise RuntimeError("reference-body encoder failed")
        body = out[:n].tobytes()
    else:
        raise InvalidInputError(f"encoder supports codec ids 0 and 1, got {codec}")
    return struct.pack("<BBHHHHI", codec, bits, w, h, count, 0, len(body)) + body + \
        struct.pack("<I", crc)


class _Positions:
    sh_degree = None

    def __init__(self, p):
        self.positions = p

    def __len__(self):
        return self.positions.shape[0]


@dataclass
class _Group:
    start: int
    frames: int
    position_bits: int
    layer_counts: list
    # per layer: list of (attr, comp, bits, rmin, rmax, {codec: payload})
    layers: list


def _encode_group(frames: list, start: int, cfg: EncodeConfig, position_bits: int,
                  codecs: Sequence[int], pool, lib) -> _Group:
    key = frames[0]
    keep = _keep_after_prune(key.opacities, cfg.prune_fraction)
    idx = keep[_significance_rank(key.take(keep), cfg.volume_weight)]
    sizes = _layer_sizes(len(idx), cfg.fractions())
    if any(s < 1 for s in sizes):
        raise InvalidInputError(f"group at frame {start}: a layer would be empty "
                                f"({len(idx)} splats across {cfg.layer_count} layers)")
    ordered = [f.take(idx) for f in frames]
    rots = [ordered[0].rotations]
    for g in ordered[1:]:
        q = g.rotations
        s = np.sign(np.sum(q * rots[-1], axis=1))
        s[s == 0] = 1.0
        rots.append(q * s[:, None])
    shdim = sh_coeff_count(key.sh_degree)
    cols = {"position": [g.positions for g in ordered], "rotation": rots,
            "scales": [g.scales for g in ordered],
            "opacity": [g.opacities[:, None] for g in ordered], "sh": [g.sh for g in ordered]}
    width = dict(_WIDTH, sh=shdim)
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    def channel(lo, hi, attr, comp, bits):
        mat = np.stack([a[lo:hi, comp] for a in cols[attr]])
        codes, rmin, rmax = _quantize(mat.ravel(), bits)
        planes = _planes(codes.reshape(mat.shape))
        return [attr, comp, bits, rmin, rmax, {c: _payload(planes, bits, c, lib) for c in codecs}]

    jobs = []
    for l in range(cfg.layer_count):
        lo, hi = int(bounds[l]), int(bounds[l + 1])
        jobs.append([pool.submit(channel, lo, hi, attr, comp,
                                 position_bits if attr == "position" else 8)
                     for attr in _ATTRS_SORTED for comp in range(width[attr])])
    layers = [[f.result() for f in js] for js in jobs]
    return _Group(start, len(frames), position_bits, sizes, layers)


class _PendingGroup:
    """A group quantised on the device, waiting for the batched range coder."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


def _gpu_quantize_group(frames: list, start: int, cfg: EncodeConfig, position_bits: int, sess):
    """_encode_group on the GPU, first half: the keyframe
    ordering (prune, significance rank, layer sizes) stays on the host; the
    frames are gathered into that order on the device, rotations
    hemisphere-aligned (pipeline.py:200-207: flip = sign(((p0 + p1) + p2) +
    p3), numpy's summation order), and every (layer, channel) is quantised
    into padded planes by gsv_quantize_channels (encode.cu)."""
    import torch

    from . import _lib
    L = _lib.load()
    key = frames[0]
    keep = _keep_after_prune(key.opacities, cfg.prune_fraction)
    idx = keep[_significance_rank(key.take(keep), cfg.volume_weight)]
    sizes = _layer_sizes(len(idx), cfg.fractions())
    if any(s < 1 for s in sizes):
        raise InvalidInputError(f"group at frame {start}: a layer would be empty "
                                f"({len(idx)} splats across {cfg.layer_count} layers)")
    shdim = sh_coeff_count(key.sh_degree)
    width = dict(_WIDTH, sh=shdim)
    col0 = {"position": 0, "rotation": 3, "scales": 7, "opacity": 10, "sh": 11}
    ncol = 11 + shdim
    dev = torch.device("cuda", sess.device)
    nf, n = len(frames), len(idx)
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    chans = []  # (layer, attr, comp, bits, lo, hi, w, h)
    for l in range(cfg.layer_count):
        lo, hi = int(bounds[l]), int(bounds[l + 1])
        w, h = _plane_shape(hi - lo)
        if max(w, h, nf) > 0xFFFF:
            raise InvalidInputError("plane run exceeds u16 geometry limits")
        for attr in _ATTRS_SORTED:
            for comp in range(width[attr]):
                chans.append((l, attr, comp, position_bits if attr == "position" else 8, lo, hi, w, h))
    with torch.cuda.stream(sess.stream):
        d_idx = torch.from_numpy(np.ascontiguousarray(idx)).to(dev)
        cols = torch.empty((ncol, nf, n), dtype=torch.float64, device=dev)  # significance order
        for t, f in enumerate(frames):
            for c0, a in ((0, f.positions), (3, f.rotations), (7, f.scales), (10, f.opacities), (11, f.sh)):
                a = torch.from_numpy(np.require(a, np.float64, ["C", "W"]).reshape(len(f), -1)).to(dev)
                cols[c0:c0 + a.shape[1], t, :] = a.index_select(0, d_idx).t()
        rot = cols[3:7]
        for t in range(1, nf):
            p = rot[:, t] * rot[:, t - 1]
            flip = torch.sign(((p[0] + p[1]) + p[2]) + p[3])
            flip[flip == 0] = 1.0
            rot[:, t] *= flip
        offs, total = [], 0
        for (_, _, _, bits, _, _, w, h) in chans:
            offs.append(total)
            total += (nf * w * h * (bits // 8) + 15) & ~15
        planes = torch.empty(max(total, 16), dtype=torch.uint8, device=dev)
        qc = (_lib.QuantChannel_t * len(chans))()
        for i, (l, attr, comp, bits, lo, hi, w, h) in enumerate(chans):
            qc[i] = _lib.QuantChannel_t(cols[col0[attr] + comp].data_ptr() + 8 * lo,
                                        planes.data_ptr() + offs[i], n, nf, hi - lo, w, h, bits, 0.0, 0.0)
        _lib.check(L.gsv_quantize_channels(sess.handle, qc, len(chans)))
    ranges = [(float(q.range_min), float(q.range_max)) for q in qc]
    return _PendingGroup(start=start, nf=nf, position_bits=position_bits, sizes=sizes, chans=chans,
                         offs=offs, planes=planes, ranges=ranges, layer_count=cfg.layer_count)


def _gpu_finish(pending: list, codecs: Sequence[int], sess) -> list:
    """Second half: every run of every pending group range-coded in ONE
    gsv_encode_runs call (runs are sequential inside, so parallelism comes
    from the number of runs: batching groups is what fills the GPU), bodies
    and raw planes read back once, payloads assembled (encode_planes,
    codec.py:166-180)."""
    import torch

    from . import _lib
    L = _lib.load()
    items = [(g, i) for g in pending for i in range(len(g.chans))]
    runs = (_lib.EncodeRun_t * max(len(items), 1))()
    h_bodies = None
    with torch.cuda.stream(sess.stream):
        if 1 in codecs and items:
            caps = [int(L.gsv_encode_body_capacity(g.nf, g.chans[i][6], g.chans[i][7], g.chans[i][3]))
                    for g, i in items]
            boffs = np.concatenate([[0], np.cumsum([(c + 15) & ~15 for c in caps])]).astype(np.int64)
            # zeroed: the copy back below reads each body's whole capacity slot
            bodies = torch.zeros(int(boffs[-1]) + 16, dtype=torch.uint8, device=sess.device)
            for k, (g, i) in enumerate(items):
                _, _, _, bits, _, _, w, h = g.chans[i]
                runs[k] = _lib.EncodeRun_t(g.planes.data_ptr() + g.offs[i], bodies.data_ptr() + int(boffs[k]),
                                           g.nf, w, h, bits, 0, 0, 0)
            t0 = time.perf_counter()
            _lib.check(L.gsv_encode_runs(sess.handle, runs, len(items)))
            if os.environ.get("GSV_DEBUG_ENC_TIMING"):  # dev: range-coder time to stderr
                print(f"[enc] range-code {len(items)} runs {1e3 * (time.perf_counter() - t0):.1f} ms",
                      file=sys.stderr)
            h_bodies = bodies.cpu().numpy()
            del bodies
        h_planes = {id(g): g.planes.cpu().numpy() for g in pending} if (0 in codecs or h_bodies is None) else {}
    out = []
    k = 0
    for g in pending:
        layers = [[] for _ in range(g.layer_count)]
        for i, (l, attr, comp, bits, lo, hi, w, h) in enumerate(g.chans):
            raw_len = g.nf * w * h * (bits // 8)
            raw = h_planes[id(g)][g.offs[i]:g.offs[i] + raw_len].tobytes() if h_planes else None
            crc = int(runs[k].checksum) if h_bodies is not None else zlib.crc32(raw) & 0xFFFFFFFF
            payloads = {}
            for c in codecs:
                if c == 0:
                    body = raw
                elif c == 1:
                    body = h_bodies[int(boffs[k]):int(boffs[k]) + int(runs[k].body_len)].tobytes()
                else:
                    raise InvalidInputError(f"encoder supports codec ids 0 and 1, got {c}")
                payloads[c] = struct.pack("<BBHHHHI", c, bits, w, h, g.nf, 0, len(body)) + body + \
                    struct.pack("<I", crc)
            layers[l].append([attr, comp, bits, g.ranges[i][0], g.ranges[i][1], payloads])
            k += 1
        out.append(_Group(g.start, g.nf, g.position_bits, g.sizes, layers))
    return out


def _encode_group_gpu(frames: list, start: int, cfg: EncodeConfig, position_bits: int,
                      codecs: Sequence[int], sess) -> _Group:
    """_encode_group on the GPU (quantise + range-code one group)."""
    return _gpu_finish([_gpu_quantize_group(frames, start, cfg, position_bits, sess)], codecs, sess)[0]


def _serialize(groups: list, codec: int, cfg: EncodeConfig, sh_degree: int, bounds) -> bytes:
    L = cfg.layer_count
    dir_size = sum(8 + 4 * L + sum(2 + 28 * len(ents) for ents in g.layers) for g in groups)
    off = 42 + dir_size
    head = [struct.pack("<4sHBBHHH6fI", b"GSV1", 1, L, sh_degree, len(groups), cfg.fps[0],
                        cfg.fps[1], *[float(b) for b in bounds], 0)]
    chunks = []
    for g in groups:
        head.append(struct.pack("<IHBB", g.start, g.frames, g.position_bits, 0))
        head.append(struct.pack(f"<{L}I", *[int(c) for c in g.layer_counts]))
        for ents in g.layers:
            head.append(struct.pack("<H", len(ents)))
            for attr, comp, bits, rmin, rmax, payloads in ents:
                p = payloads[codec]
                head.append(struct.pack("<BHBQQff", ATTRIBUTE_CODES[attr], comp, bits, off, len(p),
                                        rmin, rmax))
                chunks.append(p)
                off += len(p)
    return b"".join(head + chunks)


def encode_stream(frame_source: Callable[[], Iterable[GaussianSet]], cfg: EncodeConfig, *,
                  codecs: Sequence[int] | None = None, threads: int | None = None,
                  positions_source: Callable[[], Iterable[np.ndarray]] | None = None,
                  device=None) -> dict:
    """Encode the sequence produced by `frame_source()` (called twice: a
    statistics pass for bounds / position width / group cuts, then the encode
    pass; `positions_source`, if given, replaces the first pass with a stream
    of (N, 3) position arrays).  Returns {codec: container bytes}.

    device: None encodes on host threads; True or an api.Session quantises
    and range-codes on the GPU (_encode_group_gpu), with identical bytes."""
    from . import _lib
    lib = _lib.load()
    codecs = tuple(codecs) if codecs is not None else (int(cfg.codec),)
    mins = maxs = None
    cuts = [0]
    prev = None
    nframes = 0
    sh_degree = None
    stats_iter = positions_source() if positions_source is not None else frame_source()
    for t, f in enumerate(stats_iter):
        if isinstance(f, np.ndarray):
            f = _Positions(f)
        if len(f) == 0:
            raise InvalidInputError(f"frame {t} is empty")
        if f.sh_degree is None:
            pass
        elif sh_degree is None:
            sh_degree = f.sh_degree
        elif f.sh_degree != sh_degree:
            raise InvalidInputError("frames disagree on SH degree")
        lo, hi = f.positions.min(axis=0), f.positions.max(axis=0)
        mins = lo if mins is None else np.minimum(mins, lo)
        maxs = hi if maxs is None else np.maximum(maxs, hi)
        if t > 0 and cfg.fixed_group_length is None:
            if len(f) != len(prev):
                v = np.inf
            else:
                v = float(np.linalg.norm(f.positions - prev.positions, axis=1).mean())
            if v > cfg.motion_threshold:
                cuts.append(t)
        prev = f
        nframes += 1
    if nframes == 0:
        raise InvalidInputError("no frames to encode")
    if cfg.fixed_group_length is not None:
        cuts = list(range(0, nframes, cfg.fixed_group_length))
    extent = float((maxs - mins).max())
    if sh_degree is None:
        sh_degree = next(iter(frame_source())).sh_degree
    position_bits = 32 if (cfg.position_bits == 32 or extent > cfg.wide_extent) else 16
    ends = cuts[1:] + [nframes]
    groups = []
    threads = threads or max(1, (os.cpu_count() or 1))
    sess = None
    if device is not None and device is not False:
        from .api import Session
        sess = device if isinstance(device, Session) else Session()
    pending, pending_bytes = [], 0
    batch_bytes = int(float(os.environ.get("GSV_ENC_BATCH_GB", "8")) * 2 ** 30)
    with ThreadPoolExecutor(max_workers=threads) as pool:
        buf, gi = [], 0
        for t, f in enumerate(frame_source()):
            buf.append(f)
            if t + 1 == ends[gi]:
                if sess is not None:  # quantise now, range-code in batches of groups
                    pending.append(_gpu_quantize_group(buf, cuts[gi], cfg, position_bits, sess))
                    pending_bytes += pending[-1].planes.numel()
                    if pending_bytes > batch_bytes:
                        groups.extend(_gpu_finish(pending, codecs, sess))
                        pending, pending_bytes = [], 0
                else:
                    groups.append(_encode_group(buf, cuts[gi], cfg, position_bits, codecs, pool, lib))
                buf, gi = [], gi + 1
    if pending:
        groups.extend(_gpu_finish(pending, codecs, sess))
    bounds = (*mins.tolist(), *maxs.tolist())
    return {c: _serialize(groups, c, cfg, sh_degree, bounds) for c in codecs}


def encode_sequence_bytes(frames: Sequence[GaussianSet], cfg: EncodeConfig) -> bytes:
    """encode_sequence for in-memory frames; returns the container bytes."""
    return encode_stream(lambda: iter(frames), cfg)[int(cfg.codec)]
