"""Host-side data types mirroring the reference's dataclasses.

Same field names and semantics as the reference (paths relative to
/root/reference/pkg/src/gsv/):  GaussianSet (gaussians.py:59-149),
LayeredFrame (169-201), RigidDelta / ResidualDelta / FrameDelta
(motion.py:58-141), Camera / Image (render.py:43-162), ChannelEntry /
GroupDirectory / ContainerInfo / DecodedGroup / DecodedVideo
(container.py:44-81, 199-223), Plane / CodedPayload (quantize.py:120-148,
codec.py:58-92).  The API functions accept either these or the reference's
own objects (duck typing on the field names).
"""

from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .errors import CodecError, InvalidInputError

ATTRIBUTE_CODES = {"position": 0, "rotation": 1, "scales": 2, "opacity": 3, "sh": 4}
ATTRIBUTE_NAMES = {v: k for k, v in ATTRIBUTE_CODES.items()}


def sh_coeff_count(sh_degree: int) -> int:
    if sh_degree not in (0, 1, 2, 3):
        raise InvalidInputError(f"sh_degree must be 0..3, got {sh_degree}")
    return 3 * (sh_degree + 1) ** 2


def _frozen(a, dtype=np.float64):
    arr = np.ascontiguousarray(np.asarray(a, dtype=dtype))
    arr.flags.writeable = False
    return arr


@dataclass(frozen=True)
class GaussianSet:
    positions: np.ndarray   # (N, 3) float64
    rotations: np.ndarray   # (N, 4) float64 (w, x, y, z), not renormalised
    scales: np.ndarray      # (N, 3)
    opacities: np.ndarray   # (N,)
    sh: np.ndarray          # (N, 3*(deg+1)^2), coefficient-major RGB triples
    sh_degree: int

    def __post_init__(self):
        n = np.asarray(self.positions).shape[0]
        expected = {"positions": (n, 3), "rotations": (n, 4), "scales": (n, 3),
                    "opacities": (n,), "sh": (n, sh_coeff_count(self.sh_degree))}
        for name, shape in expected.items():
            arr = _frozen(getattr(self, name))
            if arr.shape != shape:
                raise InvalidInputError(f"{name} has shape {arr.shape}, expected {shape}")
            object.__setattr__(self, name, arr)

    def __len__(self) -> int:
        return self.positions.shape[0]

    def take(self, indices) -> "GaussianSet":
        idx = np.asarray(indices, dtype=np.int64)
        return GaussianSet(self.positions[idx], self.rotations[idx], self.scales[idx],
                           self.opacities[idx], self.sh[idx], self.sh_degree)


def concat_sets(sets: Sequence) -> GaussianSet:
    if not sets:
        raise InvalidInputError("nothing to concatenate")
    deg = sets[0].sh_degree
    if any(s.sh_degree != deg for s in sets):
        raise InvalidInputError("mixed SH degrees")
    return GaussianSet(*(np.concatenate([getattr(s, n) for s in sets]) for n in
                         ("positions", "rotations", "scales", "opacities", "sh")), deg)


@dataclass(frozen=True)
class LayeredFrame:
    layers: tuple
    layer_fractions: tuple
    volume_weight: float

    def __post_init__(self):
        if len(self.layers) < 1:
            raise InvalidInputError("at least one layer required")
        if len(self.layer_fractions) != len(self.layers):
            raise InvalidInputError("one fraction per layer required")

    @property
    def layer_count(self) -> int:
        return len(self.layers)

    @property
    def layer_sizes(self) -> tuple:
        return tuple(len(s) for s in self.layers)

    def flatten(self, up_to: int | None = None) -> GaussianSet:
        l = self.layer_count if up_to is None else up_to
        if not 1 <= l <= self.layer_count:
            raise InvalidInputError(f"layer index {l} out of range 1..{self.layer_count}")
        return concat_sets(self.layers[:l])


@dataclass(frozen=True)
class RigidDelta:
    translations: np.ndarray  # (N, 3)
    rotations: np.ndarray     # (N, 4) unit quaternions, applied on the left

    def __post_init__(self):
        t, r = _frozen(self.translations), _frozen(self.rotations)
        if t.ndim != 2 or t.shape[1] != 3 or r.shape != (t.shape[0], 4):
            raise InvalidInputError("translations must be (N,3) and rotations (N,4)")
        if not (np.all(np.isfinite(t)) and np.all(np.isfinite(r))):
            raise InvalidInputError("non-finite rigid delta")
        if np.any(np.abs(np.linalg.norm(r, axis=1) - 1.0) > 1e-6):
            raise InvalidInputError("delta rotations must be unit quaternions")
        object.__setattr__(self, "translations", t)
        object.__setattr__(self, "rotations", r)

    def __len__(self):
        return self.translations.shape[0]


@dataclass(frozen=True)
class ResidualDelta:
    d_scales: np.ndarray
    d_opacity: np.ndarray
    d_sh: np.ndarray

    def __post_init__(self):
        ds, do, dsh = _frozen(self.d_scales), _frozen(self.d_opacity), _frozen(self.d_sh)
        n = ds.shape[0]
        if ds.shape != (n, 3) or do.shape != (n,) or dsh.ndim != 2 or dsh.shape[0] != n:
            raise InvalidInputError("residual delta arrays must share length N")
        for arr in (ds, do, dsh):
            if not np.all(np.isfinite(arr)):
                raise InvalidInputError("non-finite residual delta")
        object.__setattr__(self, "d_scales", ds)
        object.__setattr__(self, "d_opacity", do)
        object.__setattr__(self, "d_sh", dsh)

    def __len__(self):
        return self.d_scales.shape[0]


@dataclass(frozen=True)
class FrameDelta:
    rigid: RigidDelta
    residual: ResidualDelta
    frame_index: int

    def __post_init__(self):
        if len(self.rigid) != len(self.residual):
            raise InvalidInputError("rigid and residual deltas must match in length")

    def __len__(self):
        return len(self.rigid)

    def prefix(self, count: int) -> "FrameDelta":
        if not 0 <= count <= len(self):
            raise InvalidInputError("prefix count out of range")
        return FrameDelta(RigidDelta(self.rigid.translations[:count], self.rigid.rotations[:count]),
                          ResidualDelta(self.residual.d_scales[:count],
                                        self.residual.d_opacity[:count],
                                        self.residual.d_sh[:count]), self.frame_index)


@dataclass(frozen=True)
class Camera:
    """Pinhole camera: x_cam = rotation @ x_world + translation."""

    rotation: np.ndarray
    translation: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float = 0.01
    background: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        r, t = _frozen(self.rotation), _frozen(self.translation)
        if r.shape != (3, 3) or t.shape != (3,):
            raise InvalidInputError("rotation must be 3x3 and translation a 3-vector")
        if self.fx <= 0 or self.fy <= 0:
            raise InvalidInputError("focal lengths must be positive")
        if self.width < 1 or self.height < 1:
            raise InvalidInputError("image dimensions must be >= 1")
        if self.near <= 0:
            raise InvalidInputError("near plane must be positive")
        object.__setattr__(self, "rotation", r)
        object.__setattr__(self, "translation", t)

    @property
    def center(self) -> np.ndarray:
        return -self.rotation.T @ self.translation

    @classmethod
    def looking_at(cls, eye, target, up=(0.0, 1.0, 0.0), *, fov_deg=60.0, width=256, height=256,
                   near=0.01, background=(0.0, 0.0, 0.0)) -> "Camera":
        eye = np.asarray(eye, dtype=np.float64)
        fwd = np.asarray(target, dtype=np.float64) - eye
        norm = np.linalg.norm(fwd)
        if norm == 0:
            raise InvalidInputError("eye and target coincide")
        fwd = fwd / norm
        right = np.cross(fwd, np.asarray(up, dtype=np.float64))
        rnorm = np.linalg.norm(right)
        if rnorm < 1e-12:
            raise InvalidInputError("up vector is parallel to the view direction")
        right /= rnorm
        down = np.cross(fwd, right)
        rot = np.stack([right, down, fwd])
        fx = width / (2.0 * math.tan(math.radians(fov_deg) / 2.0))
        return cls(rotation=rot, translation=-rot @ eye, fx=fx, fy=fx, cx=width / 2.0,
                   cy=height / 2.0, width=width, height=height, near=near,
                   background=tuple(background))

    def to_json_dict(self) -> dict:
        return {"rotation": self.rotation.tolist(), "translation": self.translation.tolist(),
                "fx": self.fx, "fy": self.fy, "cx": self.cx, "cy": self.cy,
                "width": self.width, "height": self.height, "near": self.near,
                "background": list(self.background)}

    @classmethod
    def from_json_dict(cls, d: dict) -> "Camera":
        return cls(rotation=np.asarray(d["rotation"], dtype=np.float64),
                   translation=np.asarray(d["translation"], dtype=np.float64),
                   fx=float(d["fx"]), fy=float(d["fy"]), cx=float(d["cx"]), cy=float(d["cy"]),
                   width=int(d["width"]), height=int(d["height"]),
                   near=float(d.get("near", 0.01)),
                   background=tuple(d.get("background", (0.0, 0.0, 0.0))))


def load_camera(path) -> Camera:
    with open(path, "r", encoding="utf-8") as f:
        return Camera.from_json_dict(json.load(f))


@dataclass(frozen=True)
class Splat2D:
    """A projected Gaussian ready for compositing (render.py:132-140)."""

    mean2d: np.ndarray    # (2,) pixel coordinates
    cov2d: np.ndarray     # (2, 2) symmetric positive definite, px^2
    depth: float          # camera-space z
    color: np.ndarray     # (3,) RGB in [0, 1]
    base_opacity: float


@dataclass(frozen=True)
class Image:
    """An HxWx3 float image with channels in [0, 1]."""

    pixels: np.ndarray

    def __post_init__(self):
        p = _frozen(self.pixels)
        if p.ndim != 3 or p.shape[2] != 3:
            raise InvalidInputError("pixels must be (H, W, 3)")
        object.__setattr__(self, "pixels", p)

    @property
    def width(self) -> int:
        return self.pixels.shape[1]

    @property
    def height(self) -> int:
        return self.pixels.shape[0]


@dataclass(frozen=True, order=True)
class ChannelId:
    attribute: str
    component: int

    def __str__(self) -> str:
        return f"{self.attribute}[{self.component}]"


@dataclass(frozen=True)
class ChannelEntry:
    channel: ChannelId
    bits: int
    offset: int
    size: int
    range_min: float
    range_max: float


@dataclass(frozen=True)
class GroupDirectory:
    start_frame: int
    frame_count: int
    position_bits: int
    layer_counts: tuple
    channels: tuple

    def layer_bytes(self, layer: int) -> int:
        return sum(e.size for e in self.channels[layer])

    def segment_range(self, layer: int) -> tuple:
        entries = self.channels[layer]
        start = entries[0].offset
        end = entries[-1].offset + entries[-1].size
        return start, end - start


@dataclass(frozen=True)
class ContainerInfo:
    version: int
    layer_count: int
    sh_degree: int
    fps: tuple
    bounds: tuple
    flags: int
    groups: tuple


@dataclass(frozen=True)
class DecodedGroup:
    start_frame: int
    frame_count: int
    layer_counts: tuple
    frames: tuple


@dataclass(frozen=True)
class DecodedVideo:
    layer_count: int
    decoded_layers: int
    sh_degree: int
    fps: tuple
    groups: tuple

    @property
    def frame_count(self) -> int:
        return sum(g.frame_count for g in self.groups)

    def frame(self, t: int) -> GaussianSet:
        for g in self.groups:
            if g.start_frame <= t < g.start_frame + g.frame_count:
                return g.frames[t - g.start_frame]
        raise InvalidInputError(f"frame {t} out of range 0..{self.frame_count - 1}")


@dataclass(frozen=True)
class Plane:
    samples: np.ndarray
    valid_count: int

    @property
    def width(self) -> int:
        return self.samples.shape[1]

    @property
    def height(self) -> int:
        return self.samples.shape[0]

    @property
    def bits(self) -> int:
        return self.samples.dtype.itemsize * 8


PAYLOAD_HEADER = struct.Struct("<BBHHHHI")


@dataclass(frozen=True)
class CodedPayload:
    codec_id: int
    bits: int
    width: int
    height: int
    count: int
    body: bytes
    checksum: int

    def to_bytes(self) -> bytes:
        return (PAYLOAD_HEADER.pack(self.codec_id, self.bits, self.width, self.height,
                                    self.count, 0, len(self.body))
                + self.body + struct.pack("<I", self.checksum))

    @classmethod
    def from_bytes(cls, data: bytes, offset: int = 0):
        if len(data) - offset < PAYLOAD_HEADER.size:
            raise CodecError("payload header truncated")
        codec_id, bits, w, h, count, _, length = PAYLOAD_HEADER.unpack_from(data, offset)
        body_start = offset + PAYLOAD_HEADER.size
        end = body_start + length + 4
        if len(data) < end:
            raise CodecError("payload body truncated")
        body = bytes(data[body_start:body_start + length])
        (checksum,) = struct.unpack_from("<I", data, body_start + length)
        return cls(codec_id, bits, w, h, count, body, checksum), end
