"""Helpers for reading the reference-generated fixtures in tests/golden/."""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@dataclass
class Cam:
    """Duck-typed stand-in for gsv.render.Camera (render.py:43-120)."""

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

    @classmethod
    def from_json(cls, d):
        return cls(np.asarray(d["rotation"], np.float64), np.asarray(d["translation"], np.float64),
                   float(d["fx"]), float(d["fy"]), float(d["cx"]), float(d["cy"]),
                   int(d["width"]), int(d["height"]), float(d.get("near", 0.01)),
                   tuple(d.get("background", (0.0, 0.0, 0.0))))


@lru_cache(None)
def doc():
    return json.loads((GOLDEN / "golden.json").read_text())


def container(name: str) -> bytes:
    return (GOLDEN / "containers" / f"{name}.gsv").read_bytes()


@lru_cache(None)
def renders(name: str):
    return dict(np.load(GOLDEN / "renders" / f"{name}.npz"))


def camera(scene: str, which: str) -> Cam:
    return Cam.from_json(doc()["cameras"][scene][which])


def set_sha(g) -> str:
    h = hashlib.sha256()
    for n in ("positions", "rotations", "scales", "opacities", "sh"):
        h.update(np.ascontiguousarray(getattr(g, n), dtype=np.float64).tobytes())
    return h.hexdigest()


def scene_names():
    return list(doc()["scenes"].keys())


class _NS:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def progressive_inputs():
    """(layers, deltas, camera, doc) for the reference's moving-scene case."""
    d = doc()["progressive"]
    a = renders("progressive")
    layers = []
    for li in range(d["layer_count"]):
        layers.append(_NS(**{nm: a[f"layer{li}_{nm}"] for nm in
                             ("positions", "rotations", "scales", "opacities", "sh")},
                          sh_degree=d["sh_degree"]))
    deltas = []
    for di in range(d["n_deltas"]):
        rigid = _NS(translations=a[f"delta{di}_translations"], rotations=a[f"delta{di}_rotations"])
        res = _NS(d_scales=a[f"delta{di}_d_scales"], d_opacity=a[f"delta{di}_d_opacity"],
                  d_sh=a[f"delta{di}_d_sh"])
        deltas.append(_NS(rigid=rigid, residual=res, frame_index=di + 1,
                          __len__=None))
    return layers, deltas, Cam.from_json(d["camera"]), d, a
