"""Public decode/render API, a drop-in for the reference's entry points.

Mirrors (paths relative to /root/reference/pkg/src/gsv/):
  decode_video(source, up_to_layer=None)        pipeline.py:350-359
  read_layers(source, up_to_layer)              container.py:260-310
  read_structure(f) / read_container_info(path) container.py:151-196
  decode_planes(payload)                        codec.py:226-263
  render_set(gset, cam)                         render.py:382-385
  render_progressive(frame, k, deltas, t, cam)  render.py:388-398
  reconstruct_frame(keyframe, deltas, t, k)     motion.py:218-235
with the same argument meaning, return types and exceptions.  All compute
runs in libgsv_b200.so on the GPU; torch only provides device memory and
the stream.  `DeviceVideo` is the zero-copy fast path: a decoded layer
prefix resident in HBM that renders frames into device tensors.
"""

from __future__ import annotations

import ctypes
import math
import os
import tempfile
import io
import struct
import threading
from pathlib import Path
from typing import Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, camera_struct
from .errors import CodecError, FormatError, InvalidInputError
from .types import (ATTRIBUTE_NAMES, ChannelEntry, ChannelId, CodedPayload, ContainerInfo,
                    DecodedGroup, DecodedVideo, GaussianSet, GroupDirectory, Image, Plane,
                    sh_coeff_count)

_LE = {8: np.dtype("<u1"), 16: np.dtype("<u2"), 32: np.dtype("<u4")}


# ---------------------------------------------------------------------------
# sessions
# ---------------------------------------------------------------------------
class Session:
    """A CUDA device + stream + scratch workspace inside libgsv_b200."""

    def __init__(self, device: int | None = None, stream: torch.cuda.Stream | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2509_17513_b200 needs a CUDA device (B200); none is visible")
        L = _lib.load()
        self.device = torch.cuda.current_device() if device is None else int(device)
        # high priority: a container open's upload / decode / CRC kernels get
        # SMs ahead of frame rendering on the auxiliary streams
        self.stream = stream if stream is not None else torch.cuda.Stream(device=self.device, priority=-1)
        h = ctypes.c_void_p()
        check(L.gsv_session_create(self.device, self.stream.cuda_stream, ctypes.byref(h)))
        self.handle = h
        self.lib = L

    def sync(self):
        check(self.lib.gsv_session_sync(self.handle))

    def close(self):
        if self.handle:
            self.lib.gsv_session_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


_sessions = threading.local()


def default_session() -> Session:
    dev = torch.cuda.current_device() if torch.cuda.is_available() else 0
    d = getattr(_sessions, "by_device", None)
    if d is None:
        d = _sessions.by_device = {}
    if dev not in d:
        d[dev] = Session(dev)
    return d[dev]


def _pre(s: Session) -> None:
    """Session stream waits for torch's pending work (inputs are ready)."""
    s.stream.wait_stream(torch.cuda.current_stream(s.device))


def _post(s: Session) -> None:
    """torch's stream waits for the session's work (outputs are ready)."""
    torch.cuda.current_stream(s.device).wait_stream(s.stream)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


# ---------------------------------------------------------------------------
# container structure (host only)
# ---------------------------------------------------------------------------
def _read_all(source) -> bytes:
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source)
    if isinstance(source, (str, Path)):
        return Path(source).read_bytes()
    return source.read()


def _structure_from_bytes(data: bytes) -> ContainerInfo:
    """read_structure from the container bytes: one native parse of the
    whole directory (gsv_read_directory), the reference's checks and messages."""
    L = _lib.load()
    info = _lib.Info_t()
    check(L.gsv_read_info(data, len(data), ctypes.byref(info)))
    G = int(info.group_count)
    gis = (_lib.GroupInfo_t * max(G, 1))()
    n = ctypes.c_size_t(0)
    L.gsv_read_directory(data, len(data), gis, G, None, 0, ctypes.byref(n))  # entry count
    ents = (_lib.EntryInfo_t * max(int(n.value), 1))()
    check(L.gsv_read_directory(data, len(data), gis, G, ents, int(n.value), ctypes.byref(n)))
    groups, k = [], 0
    for g in range(G):
        gi = gis[g]
        layers = []
        for l in range(info.layer_count):
            row = []
            for _ in range(gi.channel_counts[l]):
                ei = ents[k]
                k += 1
                row.append(ChannelEntry(ChannelId(ATTRIBUTE_NAMES[ei.attribute], ei.component),
                                        ei.bits, ei.offset, ei.size, float(ei.range_min),
                                        float(ei.range_max)))
            layers.append(tuple(row))
        groups.append(GroupDirectory(gi.start_frame, gi.frame_count, gi.position_bits,
                                     tuple(gi.layer_counts[:info.layer_count]), tuple(layers)))
    return ContainerInfo(info.version, info.layer_count, info.sh_degree,
                         (info.fps_num, info.fps_den), tuple(float(b) for b in info.bounds),
                         info.flags, tuple(groups))


def _read_directory(f) -> bytes:
    """Header + directory bytes from the current position of `f`, read the
    way read_structure reads them (container.py:151-191): exactly the
    header, then per group the fixed part and counts, per layer the channel
    count and its entries -- never a byte past the directory (so a prefix
    read touches no payload byte of a higher layer).  A short read returns
    the truncated bytes; the native parser then raises the reference's
    "unexpected end of container" for them."""
    out = bytearray()

    def take(n):
        chunk = f.read(n)
        out.extend(chunk)
        return len(chunk) == n

    if not take(42):
        return bytes(out)
    L, G = out[6], struct.unpack_from("<H", out, 8)[0]
    if out[:4] != b"GSV1" or struct.unpack_from("<H", out, 4)[0] != 1 or L < 1:
        return bytes(out)  # the parser raises the header's error, as the reference does
    for _ in range(G):
        if not take(8 + 4 * L):
            return bytes(out)
        for _ in range(L):
            if not take(2):
                return bytes(out)
            if not take(28 * struct.unpack_from("<H", out, len(out) - 2)[0]):
                return bytes(out)
    return bytes(out)


def _read_prefix(f, up_to_layer: int | None):
    """Read header + directory, then only the payload bytes of layers <= k
    (container.py:276-283): the returned buffer has zeros elsewhere, so no
    byte of a higher layer is ever read from `f`."""
    blob = _read_directory(f)
    info = _structure_from_bytes(blob)
    k = info.layer_count if up_to_layer is None else up_to_layer
    if not 1 <= k <= info.layer_count:
        raise InvalidInputError(f"layer {up_to_layer} out of range 1..{info.layer_count}")
    # payloads are read at their absolute offsets (read_layers seeks to
    # entry.offset, container.py:282) while the header and directory come
    # from the current position, as read_structure reads them
    L = info.layer_count
    buf = bytearray(blob)  # header + directory only (no payload bytes of any layer yet)
    for g in info.groups:
        for l in range(k):
            for e in g.channels[l]:
                f.seek(e.offset)
                chunk = f.read(e.size)
                if len(chunk) < e.size:
                    # a short read: end the buffer inside this entry so the
                    # parser raises the reference's "unexpected end" for it
                    if len(buf) > e.offset + len(chunk):
                        del buf[e.offset + len(chunk):]
                    else:
                        buf.extend(bytes(e.offset - len(buf)))
                        buf.extend(chunk)
                    return bytes(buf), info, k
                if len(buf) < e.offset + e.size:
                    buf.extend(bytes(e.offset + e.size - len(buf)))
                buf[e.offset:e.offset + e.size] = chunk
    return bytes(buf), info, k


def read_structure(f) -> ContainerInfo:
    """read_structure (container.py:151-191) for a binary file object or bytes."""
    if isinstance(f, (bytes, bytearray, memoryview)):
        return _structure_from_bytes(bytes(f))
    return _structure_from_bytes(_read_directory(f))


def read_container_info(path) -> ContainerInfo:
    with open(path, "rb") as f:
        return read_structure(f)


# ---------------------------------------------------------------------------
# decode
# ---------------------------------------------------------------------------
class DeviceVideo:
    """A layer prefix of a container decoded into HBM (gsv_video_open).

    Only the payload bytes of layers 1..k are staged; every range-coded run
    is decoded and CRC-checked on the GPU before this returns, with the
    reference's exceptions on failure.  Frames are then rendered (or
    materialised) on demand straight from the decoded code planes.
    """

    def __init__(self, source, up_to_layer: int | None = None, session: Session | None = None,
                 resident: torch.Tensor | None = None, groups: tuple | None = None,
                 info: ContainerInfo | None = None, group_list=None):
        """groups=(g0, g1): open only those groups (a streaming player's
        unit; only their bytes are staged and decoded, frames numbered from 0
        within the range).  group_list=[g, ...]: any set of groups (a rank's
        shard of the sequence), in list order, frames numbered from 0 group
        after group; works with a resident container too."""
        self.session = session or default_session()
        L = self.session.lib
        ptr = None
        if isinstance(source, torch.Tensor):
            # host (ideally pinned) uint8 tensor holding the whole container
            if source.is_cuda or source.dtype != torch.uint8:
                raise InvalidInputError("source tensor must be a host uint8 tensor")
            src = source.contiguous()
            ptr, n = src.data_ptr(), src.numel()
            want = 1 << 16
            while info is None:
                head = bytes(src[:min(n, want)].numpy())
                try:
                    info = _structure_from_bytes(head)
                    break
                except FormatError as e:
                    if "unexpected end" in str(e) and want < n:
                        want *= 4
                        continue
                    raise
            k = info.layer_count if up_to_layer is None else up_to_layer
            data = src
        elif isinstance(source, (str, Path)):
            with open(source, "rb") as f:
                data, info, k = _read_prefix(f, up_to_layer)
        elif isinstance(source, (bytes, bytearray, memoryview)):
            data = bytes(source)
            if info is None:
                info = _structure_from_bytes(data)
            k = info.layer_count if up_to_layer is None else up_to_layer
        else:
            data, info, k = _read_prefix(source, up_to_layer)
        if not 1 <= k <= info.layer_count:
            raise InvalidInputError(f"layer {up_to_layer} out of range 1..{info.layer_count}")
        self.info = info
        self._data = data
        h = ctypes.c_void_p()
        _pre(self.session)
        nbytes = data.numel() if ptr is not None else len(data)
        hptr = ptr if ptr is not None else data
        self.group_range = None
        self.group_list = None
        if group_list is not None:
            gl = [int(g) for g in group_list]
            arr = (ctypes.c_int32 * max(1, len(gl)))(*gl)
            check(L.gsv_video_open_group_list(self.session.handle, hptr, nbytes,
                                              resident.data_ptr() if resident is not None else None,
                                              k, arr, len(gl), ctypes.byref(h)))
            self.group_list = tuple(gl)
            info = ContainerInfo(info.version, info.layer_count, info.sh_degree, info.fps, info.bounds,
                                 info.flags, tuple(info.groups[g] for g in gl))
            self.info = info
        elif groups is not None:
            g0, g1 = int(groups[0]), int(groups[1])
            if resident is not None:
                raise InvalidInputError("groups= needs a host source")
            check(L.gsv_video_open_groups(self.session.handle, hptr, nbytes, k, g0, g1, ctypes.byref(h)))
            self.group_range = (g0, g1)
            info = ContainerInfo(info.version, info.layer_count, info.sh_degree, info.fps, info.bounds,
                                 info.flags, tuple(info.groups[g0:g1]))
            self.info = info
        elif resident is not None:
            check(L.gsv_video_open_resident(self.session.handle, hptr, nbytes,
                                            resident.data_ptr(), k, ctypes.byref(h)))
        else:
            check(L.gsv_video_open(self.session.handle, hptr, nbytes, k, ctypes.byref(h)))
        self.handle = h
        self.lib = L
        self.decoded_layers = L.gsv_video_decoded_layers(h)
        self.frame_count = L.gsv_video_frame_count(h)
        self.sh_degree = info.sh_degree
        self.shdim = sh_coeff_count(info.sh_degree)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.gsv_video_close(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def group_of(self, t: int) -> int:
        """Group assignment of frame t (container.py:219-223); -1 if none."""
        return self.lib.gsv_video_group_of(self.handle, int(t))

    def splat_count(self, t: int) -> int:
        g = self.group_of(t)
        if g < 0:
            raise InvalidInputError(f"frame {t} out of range 0..{self.frame_count - 1}")
        return int(self.lib.gsv_video_group_splats(self.handle, g))

    def frame_tensors(self, t: int) -> dict:
        """fp64 SoA of frame t on the device (positions, rotations, ...)."""
        n = self.splat_count(t)
        dev = torch.device("cuda", self.session.device)
        out = {"positions": torch.empty((n, 3), dtype=torch.float64, device=dev),
               "rotations": torch.empty((n, 4), dtype=torch.float64, device=dev),
               "scales": torch.empty((n, 3), dtype=torch.float64, device=dev),
               "opacities": torch.empty((n,), dtype=torch.float64, device=dev),
               "sh": torch.empty((n, self.shdim), dtype=torch.float64, device=dev)}
        _pre(self.session)
        check(self.lib.gsv_video_frame_values(self.handle, int(t), *(
            _ptr(out[k]) for k in ("positions", "rotations", "scales", "opacities", "sh"))))
        _post(self.session)
        return out

    def frame(self, t: int) -> GaussianSet:
        """DecodedVideo.frame(t) materialised on the host (fp64)."""
        d = self.frame_tensors(t)
        self.session.sync()
        return GaussianSet(*(d[k].cpu().numpy() for k in
                             ("positions", "rotations", "scales", "opacities", "sh")),
                           self.sh_degree)

    def frame_codes(self, t: int) -> torch.Tensor:
        """Decoded integer samples of frame t: (n, 11 + shdim) uint32 in slot
        order position[0..2], rotation[0..3], scales[0..2], opacity, sh[..]."""
        n = self.splat_count(t)
        out = torch.empty((n, 11 + self.shdim), dtype=torch.int32,
                          device=torch.device("cuda", self.session.device))
        _pre(self.session)
        check(self.lib.gsv_video_frame_codes(self.handle, int(t), _ptr(out)))
        _post(self.session)
        return out

    def render(self, t: int, cam, out: torch.Tensor | None = None,
               out_u8: torch.Tensor | None = None, stats: bool = False):
        """Render frame t (render_set of DecodedVideo.frame(t)) into an fp32
        (H, W, 3) device tensor; optionally also u8 (write_ppm rounding)."""
        c = camera_struct(cam)
        dev = torch.device("cuda", self.session.device)
        if out is None and out_u8 is None:
            out = torch.empty((c.height, c.width, 3), dtype=torch.float32, device=dev)
        st = _lib.RenderStats_t()
        _pre(self.session)
        check(self.lib.gsv_video_render(self.handle, int(t), ctypes.byref(c), _ptr(out),
                                        _ptr(out_u8), ctypes.byref(st)))
        _post(self.session)
        if stats:
            return out, {"n_splats": st.n_splats, "n_visible": st.n_visible,
                         "n_keys": st.n_keys, "n_keys_emitted": st.n_keys_emitted,
                         "tiles": (st.tiles_x, st.tiles_y)}
        return out

    def render_async(self, t: int, cam_struct, out: torch.Tensor | None,
                     out_u8: torch.Tensor | None = None):
        """Enqueue a render without synchronising (throughput mode).  The key
        buffer must already be large enough (render one frame with
        stats=True first); `check_overflow()` after a sync verifies it."""
        check(self.lib.gsv_video_render(self.handle, int(t), ctypes.byref(cam_struct), _ptr(out),
                                        _ptr(out_u8), ctypes.c_void_p(1)))

    def render_batch(self, frames, cam, outs=None, outs_u8=None, host_u8=None,
                     streams: int = 8, verify: bool = True):
        """Render frames[j] frame-parallel on `streams` CUDA streams.  outs /
        outs_u8: per-frame device tensors (fp32 / u8, (H, W, 3)) or None;
        host_u8: per-frame host (pinned) u8 tensors filled by D2H copies
        (complete once the session is synchronised: Session.sync or
        torch.cuda.synchronize)."""
        n = len(frames)
        c = cam if isinstance(cam, _lib.Camera_t) else camera_struct(cam)
        fr = (ctypes.c_int32 * n)(*[int(t) for t in frames])

        def arr(ts):  # output j for frame j: the first len(frames) entries
            if ts is None:
                return None
            ts = list(ts)
            if len(ts) < n:
                raise InvalidInputError(f"{len(ts)} outputs for {n} frames")
            return (ctypes.c_void_p * n)(*[None if t is None else t.data_ptr() for t in ts[:n]])
        a_out, a_u8, a_host = arr(outs), arr(outs_u8), arr(host_u8)
        _pre(self.session)
        check_ = 1 if verify else 0
        rc = self.lib.gsv_video_render_batch(self.handle, fr, n, ctypes.byref(c),
                                             ctypes.cast(a_out, ctypes.c_void_p) if a_out else None,
                                             ctypes.cast(a_u8, ctypes.c_void_p) if a_u8 else None,
                                             ctypes.cast(a_host, ctypes.c_void_p) if a_host else None,
                                             int(streams), check_)
        _lib.check(rc)
        _post(self.session)

    def project_debug(self, t: int, cam):
        """Projection outputs of frame t through the production projection
        (codes dequantised in registers from the code planes, the path
        render/render_batch run): rects (n,4; zeros when culled), fp64 depth
        (n), order (depth rank -> splat index, survivors first, stable), tile
        counts (n) and the survivor count."""
        n = self.splat_count(t)
        dev = torch.device("cuda", self.session.device)
        rects = torch.zeros((n, 4), dtype=torch.int32, device=dev)
        depth = torch.zeros((n,), dtype=torch.float64, device=dev)
        order = torch.zeros((n,), dtype=torch.int32, device=dev)
        tiles = torch.zeros((n,), dtype=torch.int32, device=dev)
        nvis = ctypes.c_int64(0)
        _pre(self.session)
        check(self.lib.gsv_video_project_debug(self.handle, int(t), ctypes.byref(camera_struct(cam)),
                                               _ptr(rects), _ptr(depth), _ptr(order), _ptr(tiles),
                                               ctypes.byref(nvis)))
        _post(self.session)
        return (rects.cpu().numpy(), depth.cpu().numpy(), order.cpu().numpy(), tiles.cpu().numpy(),
                int(nvis.value))

    def to_decoded_video(self) -> DecodedVideo:
        groups = []
        k = self.decoded_layers
        local = 0  # frames are numbered from 0 within the opened groups
        for g in self.info.groups:
            frames = tuple(self.frame(local + i) for i in range(g.frame_count))
            local += g.frame_count
            groups.append(DecodedGroup(g.start_frame, g.frame_count, tuple(g.layer_counts[:k]),
                                       frames))
        return DecodedVideo(self.info.layer_count, k, self.info.sh_degree, self.info.fps,
                            tuple(groups))


def read_layers(source, up_to_layer: int) -> DecodedVideo:
    """read_layers (container.py:260-310): decode layers 1..k of every group."""
    with DeviceVideo(source, up_to_layer) as v:
        return v.to_decoded_video()


def decode_video(source, up_to_layer: int | None = None) -> DecodedVideo:
    """decode_video (pipeline.py:350-359)."""
    if up_to_layer is None:
        if not isinstance(source, (str, Path, bytes, bytearray, memoryview)):
            pos = source.tell()
            up_to_layer = read_structure(source).layer_count
            source.seek(pos)
    return read_layers(source, up_to_layer)


def render_sequence(source, cam, up_to_layer: int | None = None, groups=None, out: torch.Tensor | None = None,
                    streams: int = 8, session: Session | None = None, info: ContainerInfo | None = None,
                    resident: torch.Tensor | None = None, outs=None, outs_u8=None, pieces=None):
    """Every frame of a container (or of the listed groups), decoded at
    prefix k and rendered, as u8 RGB in host memory: the reference's
    `decode_video(path, k)` followed by `render_set(video.frame(t), cam)` and
    write_ppm's rounding for every t (pipeline.py:350-359, render.py:382-385,
    165-169), in one pipelined call (gsv_render_sequence_host): group uploads,
    opens and frame renders with their read-back overlap, and the reference's
    exceptions are raised after the pipeline drains.

    source: container bytes or a host uint8 tensor (pinned memory makes the
    uploads asynchronous); out: optional host uint8 tensor (frames, H, W, 3),
    pinned for asynchronous read-back.  Returns `out` (frames in group-list
    order, group-major).

    resident: the whole container already in HBM (a CUDA uint8 tensor;
    nothing is uploaded); outs / outs_u8: per-frame device tensors (fp32 /
    u8, (H, W, 3)) instead of the host frames -- then `out` is only filled
    when given, and None is returned when it is not.  pieces: a list of
    (group, f0, f1) -- frames [f0, f1) of each group (a rank's shard of a
    sequence), instead of `groups`."""
    s = session or default_session()
    if isinstance(source, torch.Tensor):
        if source.is_cuda or source.dtype != torch.uint8:
            raise InvalidInputError("source tensor must be a host uint8 tensor")
        src = source.contiguous()
        hptr, nbytes = src.data_ptr(), src.numel()
        want = 1 << 16
        while info is None:  # header + directory: grow the read until the parser is satisfied
            try:
                info = _structure_from_bytes(bytes(src[:min(nbytes, want)].numpy()))
            except FormatError as e:
                if "unexpected end" in str(e) and want < nbytes:
                    want *= 4
                    continue
                raise
    else:
        src = _read_all(source)
        hptr, nbytes = src, len(src)
        if info is None:
            info = _structure_from_bytes(src)
    fb = fe = None
    if pieces is not None:
        gl = [int(p[0]) for p in pieces]
        fb = (ctypes.c_int32 * max(1, len(gl)))(*[int(p[1]) for p in pieces])
        fe = (ctypes.c_int32 * max(1, len(gl)))(*[int(p[2]) for p in pieces])
    else:
        gl = list(range(len(info.groups))) if groups is None else [int(g) for g in groups]
    for g in gl:
        if not 0 <= g < len(info.groups):
            raise InvalidInputError(f"group {g} out of range 0..{len(info.groups) - 1}")
    if pieces is not None:
        nfr = sum(max(0, int(p[2]) - int(p[1])) for p in pieces)
    else:
        nfr = sum(int(info.groups[g].frame_count) for g in gl)
    c = cam if isinstance(cam, _lib.Camera_t) else camera_struct(cam)
    H, W = int(c.height), int(c.width)
    device_out = outs is not None or outs_u8 is not None
    if out is None and not device_out:
        out = torch.empty((nfr, H, W, 3), dtype=torch.uint8, pin_memory=torch.cuda.is_available())
    host_ptrs = None
    if out is not None:
        if out.shape != (nfr, H, W, 3) or out.dtype != torch.uint8 or out.is_cuda or not out.is_contiguous():
            raise InvalidInputError(f"out must be a contiguous host uint8 tensor of shape {(nfr, H, W, 3)}")
        base, step = out.data_ptr(), H * W * 3
        host_ptrs = (ctypes.c_void_p * max(1, nfr))(*[base + j * step for j in range(nfr)])

    def dev_arr(ts, dtype):
        if ts is None:
            return None
        if len(ts) != nfr or any(t.dtype != dtype or not t.is_cuda or tuple(t.shape) != (H, W, 3) for t in ts):
            raise InvalidInputError(f"{nfr} CUDA tensors of shape {(H, W, 3)} and dtype {dtype} expected")
        return (ctypes.c_void_p * max(1, nfr))(*[t.data_ptr() for t in ts])
    a_rgb, a_u8 = dev_arr(outs, torch.float32), dev_arr(outs_u8, torch.uint8)
    if resident is not None and (not resident.is_cuda or resident.dtype != torch.uint8 or resident.numel() < nbytes):
        raise InvalidInputError("resident must be a CUDA uint8 tensor holding the whole container")
    arr = (ctypes.c_int32 * max(1, len(gl)))(*gl)
    k = -1 if up_to_layer is None else int(up_to_layer)
    written = ctypes.c_int64(0)
    _pre(s)
    check(s.lib.gsv_render_sequence(s.handle, hptr, nbytes, resident.data_ptr() if resident is not None else None,
                                    k, arr, len(gl), fb, fe, ctypes.byref(c), a_rgb, a_u8, host_ptrs, int(streams),
                                    ctypes.byref(written)))
    _post(s)
    return out


def decode_planes(payload) -> list:
    """decode_planes (codec.py:226-263) on the GPU: list of Plane."""
    blob = payload.to_bytes() if hasattr(payload, "to_bytes") else bytes(payload)
    s = default_session()
    n = max(1, int(payload.count) * int(payload.width) * int(payload.height))
    out = np.zeros(n, np.uint32)
    hdr = np.zeros(5, np.int32)
    check(s.lib.gsv_decode_payload_host(s.handle, blob, len(blob), out.ctypes.data, out.size,
                                        hdr.ctypes.data))
    bits = int(payload.bits)
    arr = out[:int(payload.count) * int(payload.width) * int(payload.height)].astype(_LE[bits])
    arr = arr.reshape(int(payload.count), int(payload.height), int(payload.width))
    planes = []
    for i in range(arr.shape[0]):
        s_ = arr[i].copy()
        s_.flags.writeable = False
        planes.append(Plane(samples=s_, valid_count=arr.shape[1] * arr.shape[2]))
    return planes


# ---------------------------------------------------------------------------
# render
# ---------------------------------------------------------------------------
def _soa_to_device(gset, dev):
    return [torch.from_numpy(np.ascontiguousarray(np.asarray(getattr(gset, k), dtype=np.float64)))
            .to(dev) for k in ("positions", "rotations", "scales", "opacities", "sh")]


def render_soa_tensors(tensors, sh_degree: int, cam, session: Session | None = None,
                       out: torch.Tensor | None = None, stats: bool = False):
    """Render device fp64 SoA tensors; returns an fp32 (H, W, 3) device tensor."""
    s = session or default_session()
    c = camera_struct(cam)
    n = int(tensors[0].shape[0])
    if out is None:
        out = torch.empty((c.height, c.width, 3), dtype=torch.float32,
                          device=torch.device("cuda", s.device))
    st = _lib.RenderStats_t()
    _pre(s)
    check(s.lib.gsv_render_soa(s.handle, n, int(sh_degree), *(_ptr(t) for t in tensors),
                               ctypes.byref(c), _ptr(out), None, ctypes.byref(st)))
    _post(s)
    if stats:
        return out, {"n_splats": st.n_splats, "n_visible": st.n_visible, "n_keys": st.n_keys,
                     "n_keys_emitted": st.n_keys_emitted, "tiles": (st.tiles_x, st.tiles_y)}
    return out


def render(splats, cam) -> Image:
    """render (render.py:359-379): composite projected splats on the GPU;
    depth order is stable (ties keep input order); no splats -> background."""
    if not splats:
        bg = np.asarray(cam.background, dtype=np.float64)
        return Image(pixels=np.tile(bg, (cam.height, cam.width, 1)))
    s = default_session()
    dev = torch.device("cuda", s.device)
    cols = [np.stack([np.asarray(sp.mean2d, np.float64) for sp in splats]),
            np.stack([np.asarray(sp.cov2d, np.float64).reshape(4) for sp in splats]),
            np.array([float(sp.depth) for sp in splats]),
            np.stack([np.asarray(sp.color, np.float64) for sp in splats]),
            np.array([float(sp.base_opacity) for sp in splats])]
    t = [torch.from_numpy(np.ascontiguousarray(c)).to(dev) for c in cols]
    c = camera_struct(cam)
    out = torch.empty((c.height, c.width, 3), dtype=torch.float32, device=dev)
    _pre(s)
    check(s.lib.gsv_render_splats2d(s.handle, len(splats), *(_ptr(x) for x in t), ctypes.byref(c),
                                    _ptr(out), None, None))
    _post(s)
    return Image(pixels=out.cpu().numpy().astype(np.float64))


PSNR_CAP = 99.0  # metrics.py:24


def psnr(gt, pred) -> float:
    """psnr (metrics.py:31-38): 10*log10(1/MSE) over all channels, capped at
    99 dB.  Images or device/host tensors; the squared-difference sum runs on
    the GPU in fp64."""
    a = gt.pixels if isinstance(gt, Image) else gt
    b = pred.pixels if isinstance(pred, Image) else pred
    if tuple(a.shape) != tuple(b.shape):
        raise InvalidInputError("image dimensions differ")
    s = default_session()
    dev = torch.device("cuda", s.device)

    def dev_t(x):
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
        return t.to(dev).contiguous()
    ta, tb = dev_t(a), dev_t(b)
    if ta.dtype != tb.dtype or ta.dtype not in (torch.float32, torch.float64):
        ta, tb = ta.to(torch.float64), tb.to(torch.float64)
    out = ctypes.c_double(0.0)
    _pre(s)
    check(s.lib.gsv_sqdiff(s.handle, _ptr(ta), _ptr(tb), ta.numel(), 1 if ta.dtype == torch.float64 else 0,
                           ctypes.byref(out)))
    _post(s)
    n = ta.numel()
    mse = out.value / n if n else 0.0
    if mse == 0.0:
        return PSNR_CAP
    return min(10.0 * math.log10(1.0 / mse), PSNR_CAP)


def _dev_pair(gt, pred, s):
    a = gt.pixels if isinstance(gt, Image) else gt
    b = pred.pixels if isinstance(pred, Image) else pred
    if tuple(a.shape) != tuple(b.shape):
        raise InvalidInputError("image dimensions differ")
    dev = torch.device("cuda", s.device)

    def dev_t(x):
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
        return t.to(dev).contiguous()
    ta, tb = dev_t(a), dev_t(b)
    if ta.dtype != tb.dtype or ta.dtype not in (torch.float32, torch.float64):
        ta, tb = ta.to(torch.float64), tb.to(torch.float64)
    return ta, tb


def ssim(gt, pred) -> float:
    """ssim (metrics.py:48-65): mean SSIM of the channel-mean images, 11x11
    Gaussian window (sigma 1.5) over valid positions; computed on the GPU."""
    s = default_session()
    ta, tb = _dev_pair(gt, pred, s)
    if ta.dim() != 3 or ta.shape[2] != 3:
        raise InvalidInputError("pixels must be (H, W, 3)")
    H, W = int(ta.shape[0]), int(ta.shape[1])
    if H < 11 or W < 11:
        raise InvalidInputError("image smaller than the SSIM window")
    out = ctypes.c_double(0.0)
    _pre(s)
    check(s.lib.gsv_ssim(s.handle, _ptr(ta), _ptr(tb), H, W, 1 if ta.dtype == torch.float64 else 0,
                         ctypes.byref(out)))
    _post(s)
    return float(out.value)


def d_ssim(gt, pred) -> float:
    """d_ssim (metrics.py:68-70): (1 - SSIM) / 2."""
    return (1.0 - ssim(gt, pred)) / 2.0


def analyze_rd(paths, cam, gt_frames, layer: int | None = None):
    """The measurement loop of cli.cmd_analyze (cli.py:147-162) on the GPU:
    for each container, decode layers 1..layer, render every frame and take
    its PSNR against gt_frames[t] without bringing images to the host.
    Returns [(rate MB/frame, mean PSNR dB)] sorted by rate, the RdPoint
    inputs (metrics.py:74-88)."""
    s = default_session()
    dev = torch.device("cuda", s.device)
    gts = [g.to(dev) if isinstance(g, torch.Tensor) else
           torch.from_numpy(np.ascontiguousarray(np.asarray(g.pixels if isinstance(g, Image) else g)))
           .to(dev) for g in gt_frames]
    c = camera_struct(cam)
    out = torch.empty((c.height, c.width, 3), dtype=torch.float32, device=dev)
    points = []
    for path in paths:
        with DeviceVideo(path, layer) as v:
            k = v.decoded_layers
            payload = sum(e.size for g in v.info.groups for l in range(k) for e in g.channels[l])
            vals = []
            for t in range(v.frame_count):
                v.render(t, cam, out=out)
                vals.append(psnr(gts[t], out.to(gts[t].dtype)))
            points.append((payload / v.frame_count / 1e6, float(np.mean(vals))))
    points.sort(key=lambda p: p[0])
    return points


def _atomic_write(path, blob: bytes) -> None:
    """splatio._atomic_write (splatio.py:107-117)."""
    path = Path(path)
    fd, tmp = tempfile.mkstemp(dir=path.parent or ".", prefix=path.name + ".")
    try:
        with os.fdopen(fd, "wb") as f:
            f.write(blob)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def write_ppm(img: Image, path) -> None:
    """write_ppm (render.py:165-169): 8-bit binary PPM (P6)."""
    u8 = np.clip(np.floor(img.pixels * 255.0 + 0.5), 0, 255).astype(np.uint8)
    header = f"P6\n{img.width} {img.height}\n255\n".encode()
    _atomic_write(path, header + u8.tobytes())


def write_raw_floats(img: Image, path) -> None:
    """write_raw_floats (render.py:172-178): lossless .npy dump."""
    import io
    buf = io.BytesIO()
    np.save(buf, img.pixels)
    _atomic_write(path, buf.getvalue())


def load_raw_floats(path) -> Image:
    return Image(pixels=np.load(path))


def render_set(gset, cam) -> Image:
    """render_set (render.py:382-385)."""
    s = default_session()
    dev = torch.device("cuda", s.device)
    img = render_soa_tensors(_soa_to_device(gset, dev), gset.sh_degree, cam, s)
    return Image(pixels=img.cpu().numpy().astype(np.float64))


def _fold_device(t_list, deltas, count, shdim, s: Session):
    dev = torch.device("cuda", s.device)
    keep = []
    for d in deltas:
        if len(d.rigid.translations) < count:
            raise InvalidInputError("delta shorter than the requested layer prefix")
        arrs = [torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)[:count]))
                .to(dev) for a in (d.rigid.translations, d.rigid.rotations, d.residual.d_scales,
                                   d.residual.d_opacity, d.residual.d_sh)]
        if arrs[4].shape[1] != shdim:
            raise InvalidInputError("d_sh width does not match the set's SH degree")
        keep.append(arrs)
    nd = len(keep)
    if nd == 0 or count == 0:
        return
    P = ctypes.c_void_p * nd
    tabs = [P(*[k[j].data_ptr() for k in keep]) for j in range(5)]
    _pre(s)
    check(s.lib.gsv_fold_deltas(s.handle, count, shdim, *(x.data_ptr() for x in t_list), nd,
                                *[ctypes.cast(tb, ctypes.c_void_p) for tb in tabs]))
    _post(s)


def _flatten(keyframe, up_to_layer):
    layers = keyframe.layers
    k = len(layers) if up_to_layer is None else up_to_layer
    if not 1 <= k <= len(layers):
        raise InvalidInputError(f"layer index {k} out of range 1..{len(layers)}")
    return layers[:k]


def reconstruct_frame_tensors(group_keyframe, deltas: Sequence, t: int, up_to_layer=None,
                              session: Session | None = None):
    """reconstruct_frame on the device: returns (tensors, sh_degree)."""
    s = session or default_session()
    if not 0 <= t <= len(deltas):
        raise InvalidInputError(f"frame index {t} out of range 0..{len(deltas)}")
    layers = _flatten(group_keyframe, up_to_layer)
    dev = torch.device("cuda", s.device)
    parts = [_soa_to_device(l, dev) for l in layers]
    tensors = [torch.cat([p[i] for p in parts]).contiguous() for i in range(5)]
    deg = layers[0].sh_degree
    _fold_device(tensors, list(deltas[:t]), int(tensors[0].shape[0]), sh_coeff_count(deg), s)
    return tensors, deg


def reconstruct_frame(group_keyframe, deltas: Sequence, t: int, up_to_layer=None) -> GaussianSet:
    """reconstruct_frame (motion.py:218-235)."""
    tensors, deg = reconstruct_frame_tensors(group_keyframe, deltas, t, up_to_layer)
    return GaussianSet(*(x.cpu().numpy() for x in tensors), deg)


def render_progressive(frame, up_to_layer: int, deltas, t: int, cam) -> Image:
    """render_progressive (render.py:388-398)."""
    if not 1 <= up_to_layer <= len(frame.layers):
        raise InvalidInputError(f"layer {up_to_layer} out of range 1..{len(frame.layers)}")
    tensors, deg = reconstruct_frame_tensors(frame, deltas, t, up_to_layer)
    img = render_soa_tensors(tensors, deg, cam)
    return Image(pixels=img.cpu().numpy().astype(np.float64))


def project_debug(gset, cam, session: Session | None = None):
    """Projection outputs for parity checks: rects (n,4; zeros when culled),
    depth (n), order (depth-rank -> splat index, survivors first), tile
    counts (n) and the survivor count."""
    s = session or default_session()
    dev = torch.device("cuda", s.device)
    tensors = _soa_to_device(gset, dev)
    n = int(tensors[0].shape[0])
    rects = torch.zeros((n, 4), dtype=torch.int32, device=dev)
    depth = torch.zeros((n,), dtype=torch.float64, device=dev)
    order = torch.zeros((n,), dtype=torch.int32, device=dev)
    tiles = torch.zeros((n,), dtype=torch.int32, device=dev)
    nvis = ctypes.c_int64(0)
    _pre(s)
    check(s.lib.gsv_project_debug(s.handle, n, int(gset.sh_degree), *(_ptr(t) for t in tensors),
                                  ctypes.byref(camera_struct(cam)), _ptr(rects), _ptr(depth),
                                  _ptr(order), _ptr(tiles), ctypes.byref(nvis)))
    _post(s)
    return (rects.cpu().numpy(), depth.cpu().numpy(), order.cpu().numpy(), tiles.cpu().numpy(),
            int(nvis.value))
