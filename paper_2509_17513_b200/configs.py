"""BASELINE.json's five benchmark configurations and their
cameras, shared by bench.py and the parity tests.

Groups are temporal motion groups (a keyframe plus the frames up to the next
burst, motion.py:203-215): a burst every `group_len` frames forces the cuts.
Config 1's "8 motion groups" over 4 frames is unsatisfiable under the
reference's semantics, so `c1` is the literal 4-frame case in 2
groups and `c1g8` the 8-group variant (16 frames, a burst every 2 frames).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .synth import SceneSpec, benchmark_spec
from .types import Camera


@dataclass(frozen=True)
class Config:
    name: str
    gaussians: int
    layers: int
    frames: int
    group_len: int
    width: int
    height: int
    seed: int
    views: int = 1
    desc: str = ""

    @property
    def groups(self) -> int:
        return -(-self.frames // self.group_len)

    def spec(self, frames: int | None = None) -> SceneSpec:
        """The generator recipe (synth.benchmark_spec); `frames` truncates the
        sequence (a prefix of the same frames: the generator is sequential)."""
        return benchmark_spec(self.gaussians, frames or self.frames, self.group_len)

    def cameras(self) -> list:
        if self.views > 1:
            return ring_cameras(self.width, self.height, self.views)
        return [axis_camera(self.width, self.height)]


CONFIGS = {
    "c1": Config("c1", 50_000, 2, 4, 2, 512, 512, 1001,
                 desc="config1: 50k Gaussians, 2 layers, 4 frames (2 groups), 512x512"),
    "c1g8": Config("c1g8", 50_000, 2, 16, 2, 512, 512, 1001,
                   desc="config1 8-group variant: 50k Gaussians, 2 layers, 16 frames (8 groups), 512x512"),
    "c2": Config("c2", 300_000, 6, 300, 30, 1920, 1080, 1002,
                 desc="config2: 300k Gaussians, 6 layers, 300 frames (10 groups), 1080p, single camera"),
    "c3": Config("c3", 1_000_000, 6, 512, 2, 1920, 1080, 1003,
                 desc="config3: 1M Gaussians, 6 layers, 512 frames (256 adaptive groups), 1080p"),
    "c4": Config("c4", 500_000, 6, 300, 30, 1920, 1080, 1004, views=16,
                 desc="config4: 500k Gaussians, 6 layers, 300 frames (10 groups), 16 ring cameras, 1080p"),
    "c5": Config("c5", 3_000_000, 6, 600, 30, 3840, 2160, 1005,
                 desc="config5: 3M Gaussians, 6 layers, 600 frames (20 groups), 3840x2160"),
}


def axis_camera(width: int, height: int) -> Camera:
    """looking_at((0, 0, -2.5)) -> origin, 60 deg: the axis view
    (about 30% of the splats tie exactly in fp64 depth)."""
    return Camera.looking_at(eye=(0.0, 0.0, -2.5), target=(0.0, 0.0, 0.0), fov_deg=60.0,
                             width=width, height=height, near=0.01)


def oblique_camera(width: int, height: int) -> Camera:
    """The second parity view of SURVEY 8(d): eye (1.3, 0.9, -1.9)."""
    return Camera.looking_at(eye=(1.3, 0.9, -1.9), target=(0.0, 0.0, 0.0), fov_deg=60.0,
                             width=width, height=height, near=0.01)


def ring_cameras(width: int, height: int, views: int = 16) -> list:
    """Config 4: looking_at cameras on a radius-2.5 ring,
    22.5 deg steps, elevation +-10 deg alternating, 60 deg fov."""
    cams = []
    for v in range(views):
        az = math.radians(22.5 * v)
        el = math.radians(10.0 if v % 2 == 0 else -10.0)
        eye = (2.5 * math.cos(el) * math.sin(az), 2.5 * math.sin(el), -2.5 * math.cos(el) * math.cos(az))
        cams.append(Camera.looking_at(eye=eye, target=(0.0, 0.0, 0.0), fov_deg=60.0,
                                      width=width, height=height, near=0.01))
    return cams
