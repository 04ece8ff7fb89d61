"""Segment-fed progressive decode.

The reference streams a container as one segment per (group, layer): the
bytes of that layer's payloads, contiguous in the container
(container.py:65-70 `segment_range`), described by a JSON manifest
(container.py:313-442).  Its client checks each fetched segment with
`_decode_segment` (streaming.py:212-223) and never renders.  Here segments
feed the GPU decode-and-render path as they arrive:

* `Manifest` / `emit_manifest` mirror the reference's manifest (same JSON
  bytes, tests/test_streaming.py pins them against the reference fixture);
* `segment(container, g, l)` cuts a segment like the reference server;
* `decode_segment(blob, manifest, g, l)` is `_decode_segment` with the
  payloads decoded on the GPU (same StreamError / CodecError messages);
* `SegmentVideo` accumulates segments; once layers 1..k of a group are
  present, the group is rebuilt as a one-group k-layer container from the
  manifest's directory data and decoded by the same C-ABI path as a whole
  container (`DeviceVideo`: one launch for all range-coded runs, CRC of
  every run), and frames of that group render at prefix k.

HTTP fetching, retries and bandwidth estimation (the reference's
client_play / server) are networking and stay out of scope.
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass

import numpy as np

from .errors import InvalidInputError, StreamError
from .types import ATTRIBUTE_CODES, CodedPayload

VERSION = 1
_HEADER = struct.Struct("<4sHBBHHH6fI")
_GROUP_FIXED = struct.Struct("<IHBB")
_CHANNEL_ENTRY = struct.Struct("<BHBQQff")


@dataclass(frozen=True)
class ManifestChannel:
    attribute: str
    component: int
    bits: int
    range_min: float
    range_max: float


@dataclass(frozen=True)
class ManifestGroup:
    start: int
    frames: int
    gauss_counts: tuple
    position_bits: int
    layer_bytes: tuple
    cum_bytes: tuple
    channels: tuple  # per layer: tuple[ManifestChannel]


@dataclass(frozen=True)
class Manifest:
    """container.Manifest (container.py:334-418)."""

    version: int
    layers: int
    fps: tuple
    sh_degree: int
    url: str
    groups: tuple

    def __post_init__(self):
        for g in self.groups:
            if any(b2 < b1 for b1, b2 in zip(g.cum_bytes, g.cum_bytes[1:])):
                raise InvalidInputError("cumulative layer sizes must be non-decreasing")

    @property
    def frame_count(self) -> int:
        return sum(g.frames for g in self.groups)

    def cum_bytes_per_frame(self, layer: int, group: int | None = None) -> float:
        if not 1 <= layer <= self.layers:
            raise InvalidInputError(f"layer {layer} out of range 1..{self.layers}")
        if group is None:
            return sum(g.cum_bytes[layer - 1] for g in self.groups) / self.frame_count
        g = self.groups[group]
        return g.cum_bytes[layer - 1] / g.frames

    def to_json_dict(self) -> dict:
        return {
            "version": self.version, "layers": self.layers, "fps": list(self.fps),
            "sh_degree": self.sh_degree, "url": self.url,
            "groups": [{
                "start": g.start, "frames": g.frames, "gauss_counts": list(g.gauss_counts),
                "position_bits": g.position_bits, "layer_bytes": list(g.layer_bytes),
                "cum_bytes": list(g.cum_bytes),
                "channels": [[{"attr": c.attribute, "comp": c.component, "bits": c.bits,
                               "min": c.range_min, "max": c.range_max} for c in layer]
                             for layer in g.channels],
            } for g in self.groups],
        }

    def to_json_bytes(self) -> bytes:
        return json.dumps(self.to_json_dict(), separators=(",", ":")).encode()

    @classmethod
    def from_json_dict(cls, d: dict) -> "Manifest":
        groups = tuple(ManifestGroup(
            start=int(g["start"]), frames=int(g["frames"]),
            gauss_counts=tuple(int(x) for x in g["gauss_counts"]),
            position_bits=int(g["position_bits"]),
            layer_bytes=tuple(int(x) for x in g["layer_bytes"]),
            cum_bytes=tuple(int(x) for x in g["cum_bytes"]),
            channels=tuple(tuple(ManifestChannel(c["attr"], int(c["comp"]), int(c["bits"]),
                                                 float(c["min"]), float(c["max"]))
                                 for c in layer) for layer in g["channels"]))
            for g in d["groups"])
        return cls(version=int(d["version"]), layers=int(d["layers"]),
                   fps=(int(d["fps"][0]), int(d["fps"][1])), sh_degree=int(d["sh_degree"]),
                   url=str(d["url"]), groups=groups)

    @classmethod
    def from_json_bytes(cls, data: bytes) -> "Manifest":
        return cls.from_json_dict(json.loads(data.decode()))


def _info(container):
    from .api import read_structure
    return read_structure(container)


def emit_manifest(container: bytes, url: str = "scene.gsv") -> Manifest:
    """emit_manifest (container.py:421-442) from container bytes."""
    info = _info(container)
    groups = []
    for g in info.groups:
        layer_bytes = tuple(sum(e.size for e in g.channels[l]) for l in range(info.layer_count))
        cum = tuple(int(x) for x in np.cumsum(layer_bytes))
        channels = tuple(tuple(ManifestChannel(e.channel.attribute, e.channel.component, e.bits,
                                               e.range_min, e.range_max) for e in layer)
                         for layer in g.channels)
        groups.append(ManifestGroup(start=g.start_frame, frames=g.frame_count,
                                    gauss_counts=tuple(g.layer_counts), position_bits=g.position_bits,
                                    layer_bytes=layer_bytes, cum_bytes=cum, channels=channels))
    return Manifest(version=VERSION, layers=info.layer_count, fps=tuple(info.fps),
                    sh_degree=info.sh_degree, url=url, groups=tuple(groups))


def segment(container: bytes, group: int, layer: int) -> bytes:
    """Bytes of one (group, layer) segment: GroupDirectory.segment_range
    (container.py:65-70) of layer `layer` (1-based)."""
    info = _info(container)
    if not 0 <= group < len(info.groups):
        raise InvalidInputError(f"group {group} out of range")
    if not 1 <= layer <= info.layer_count:
        raise InvalidInputError(f"layer {layer} out of range 1..{info.layer_count}")
    ents = info.groups[group].channels[layer - 1]
    start, end = ents[0].offset, ents[-1].offset + ents[-1].size
    return bytes(container[start:end])


def parse_payload_stream(blob: bytes) -> list:
    """codec.parse_payload_stream (codec.py:95-102): (payload, raw bytes) pairs."""
    out, off = [], 0
    while off < len(blob):
        p, end = CodedPayload.from_bytes(blob, off)
        out.append((p, bytes(blob[off:end])))
        off = end
    return out


def decode_segment(blob: bytes, manifest: Manifest, group: int, layer: int) -> None:
    """_decode_segment (streaming.py:212-223): payload count against the
    manifest, then every payload decoded (GPU) and dequantized."""
    from .api import decode_planes
    payloads = parse_payload_stream(blob)
    channels = manifest.groups[group].channels[layer - 1]
    if len(payloads) != len(channels):
        raise StreamError(f"segment g={group} l={layer}: expected "
                          f"{len(channels)} payloads, got {len(payloads)}")
    n = manifest.groups[group].gauss_counts[layer - 1]
    for (payload, _), ch in zip(payloads, channels):
        top = float((1 << ch.bits) - 1) if ch.bits < 64 else float(2 ** 64 - 1)
        for p in decode_planes(payload):
            codes = np.asarray(p.samples).reshape(-1)[:n].astype(np.float64)
            if codes.size < n:
                raise InvalidInputError(f"plane has {codes.size} samples, need {n}")
            _ = ch.range_min + codes / top * (ch.range_max - ch.range_min)


def segment_container(manifest: Manifest, group: int, segments: dict) -> bytes:
    """A one-group container of layers 1..k (k = len(segments), segments[l]
    for l = 1..k) rebuilt from the manifest's directory data, in the layout
    of write_container (container.py:103-148); start frame 0."""
    g = manifest.groups[group]
    k = len(segments)
    if k < 1 or any(l not in segments for l in range(1, k + 1)):
        raise InvalidInputError("segments must cover layers 1..k")
    layers = []
    for l in range(1, k + 1):
        payloads = parse_payload_stream(segments[l])
        chans = g.channels[l - 1]
        if len(payloads) != len(chans):
            raise StreamError(f"segment g={group} l={l}: expected {len(chans)} payloads, "
                              f"got {len(payloads)}")
        layers.append(list(zip(chans, (raw for _, raw in payloads))))
    dir_size = _GROUP_FIXED.size + 4 * k + sum(2 + _CHANNEL_ENTRY.size * len(e) for e in layers)
    off = _HEADER.size + dir_size
    out = [_HEADER.pack(b"GSV1", VERSION, k, manifest.sh_degree, 1, manifest.fps[0], manifest.fps[1],
                        *([0.0] * 6), 0),
           _GROUP_FIXED.pack(0, g.frames, g.position_bits, 0),
           struct.pack(f"<{k}I", *g.gauss_counts[:k])]
    chunks = []
    for ents in layers:
        out.append(struct.pack("<H", len(ents)))
        for ch, raw in ents:
            out.append(_CHANNEL_ENTRY.pack(ATTRIBUTE_CODES[ch.attribute], ch.component, ch.bits, off,
                                           len(raw), ch.range_min, ch.range_max))
            chunks.append(raw)
            off += len(raw)
    return b"".join(out + chunks)


class SegmentVideo:
    """Progressive player state: add (group, layer) segments in any order;
    frames of a group render with its contiguous prefix 1..k of layers."""

    def __init__(self, manifest: Manifest, session=None):
        self.manifest = manifest
        self.session = session
        self._segs = [dict() for _ in manifest.groups]
        self._videos = {}  # group -> (k, DeviceVideo)

    def add_segment(self, group: int, layer: int, blob: bytes) -> None:
        if not 0 <= group < len(self.manifest.groups):
            raise InvalidInputError(f"group {group} out of range")
        if not 1 <= layer <= self.manifest.layers:
            raise InvalidInputError(f"layer {layer} out of range 1..{self.manifest.layers}")
        payloads = parse_payload_stream(blob)
        want = len(self.manifest.groups[group].channels[layer - 1])
        if len(payloads) != want:
            raise StreamError(f"segment g={group} l={layer}: expected {want} payloads, "
                              f"got {len(payloads)}")
        self._segs[group][layer] = bytes(blob)

    def layers_ready(self, group: int) -> int:
        k = 0
        while k + 1 in self._segs[group]:
            k += 1
        return k

    def group_of(self, t: int) -> int:
        for gi, g in enumerate(self.manifest.groups):
            if g.start <= t < g.start + g.frames:
                return gi
        raise InvalidInputError(f"frame {t} out of range 0..{self.manifest.frame_count - 1}")

    def video(self, group: int):
        """DeviceVideo of the group at its ready prefix (decoded once per k)."""
        from .api import DeviceVideo
        k = self.layers_ready(group)
        if k == 0:
            raise StreamError(f"group {group}: base layer not received")
        cached = self._videos.get(group)
        if cached and cached[0] == k:
            return cached[1]
        if cached:
            cached[1].close()
        blob = segment_container(self.manifest, group, {l: self._segs[group][l] for l in range(1, k + 1)})
        v = DeviceVideo(blob, k, session=self.session)
        self._videos[group] = (k, v)
        return v

    def render(self, t: int, cam, out=None):
        """Frame t (absolute) with the layers received so far for its group:
        an fp32 (H, W, 3) device tensor."""
        gi = self.group_of(t)
        return self.video(gi).render(t - self.manifest.groups[gi].start, cam, out=out)

    def frame(self, t: int):
        gi = self.group_of(t)
        return self.video(gi).frame(t - self.manifest.groups[gi].start)

    def close(self):
        for _, v in self._videos.values():
            v.close()
        self._videos.clear()
