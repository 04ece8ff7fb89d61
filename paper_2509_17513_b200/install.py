"""Rebind a live `gsv` (the reference package) onto the B200 path.

`gsv.cli` binds names at import (cli.py:23-25), so both the defining
modules and the CLI module are patched.  Results are converted
to the reference's own dataclasses, so callers see exactly the types they
expect; exceptions are the reference's classes (errors.py is shared).
"""

from __future__ import annotations


def install(verbose: bool = False) -> dict:
    import importlib

    import gsv  # noqa: F401  (the reference must be importable)

    # by module path: `gsv.render` as an attribute is the render() function
    # the package re-exports, not the submodule
    def mod(name):
        return importlib.import_module("gsv." + name)
    gcli, gcodec, gcont = mod("cli"), mod("codec"), mod("container")
    ggauss, gmetrics, gmotion = mod("gaussians"), mod("metrics"), mod("motion")
    gpipe, gquant, grender = mod("pipeline"), mod("quantize"), mod("render")

    from . import api

    def _set(s):
        return ggauss.GaussianSet(positions=s.positions, rotations=s.rotations, scales=s.scales,
                                  opacities=s.opacities, sh=s.sh, sh_degree=s.sh_degree)

    def _video(v):
        groups = tuple(gcont.DecodedGroup(start_frame=g.start_frame, frame_count=g.frame_count,
                                          layer_counts=tuple(g.layer_counts),
                                          frames=tuple(_set(f) for f in g.frames))
                       for g in v.groups)
        return gcont.DecodedVideo(layer_count=v.layer_count, decoded_layers=v.decoded_layers,
                                  sh_degree=v.sh_degree, fps=tuple(v.fps), groups=groups)

    def decode_video(source, up_to_layer=None):
        return _video(api.decode_video(source, up_to_layer))

    def read_layers(source, up_to_layer):
        return _video(api.read_layers(source, up_to_layer))

    def decode_planes(payload):
        return [gquant.Plane(samples=p.samples, valid_count=p.valid_count)
                for p in api.decode_planes(payload)]

    def render_set(gset, cam):
        return grender.Image(pixels=api.render_set(gset, cam).pixels)

    def render_progressive(frame, up_to_layer, deltas, t, cam):
        return grender.Image(pixels=api.render_progressive(frame, up_to_layer, deltas, t,
                                                           cam).pixels)

    def reconstruct_frame(group_keyframe, deltas, t, up_to_layer=None):
        return _set(api.reconstruct_frame(group_keyframe, deltas, t, up_to_layer))

    def render(splats, cam):
        return grender.Image(pixels=api.render(splats, cam).pixels)

    def psnr(gt, pred):
        return api.psnr(gt.pixels, pred.pixels)

    patches = {
        (gpipe, "decode_video"): decode_video, (gcli, "decode_video"): decode_video,
        (gcont, "read_layers"): read_layers, (gpipe, "read_layers"): read_layers,
        (gcodec, "decode_planes"): decode_planes, (gcont, "decode_planes"): decode_planes,
        (grender, "render_set"): render_set, (gcli, "render_set"): render_set,
        (grender, "render_progressive"): render_progressive,
        (gmotion, "reconstruct_frame"): reconstruct_frame,
        (grender, "reconstruct_frame"): reconstruct_frame,
        (grender, "render"): render,
        (gmetrics, "psnr"): psnr, (gcli, "psnr"): psnr,
    }
    old = {}
    for (mod, name), fn in patches.items():
        if hasattr(mod, name):
            old[(mod.__name__, name)] = getattr(mod, name)
            setattr(mod, name, fn)
    for name in ("decode_video", "read_layers", "decode_planes", "render_set",
                 "render_progressive", "reconstruct_frame", "render", "psnr"):
        if hasattr(gsv, name):
            setattr(gsv, name, locals()[name])
    if verbose:
        print(f"gsv: {len(old)} entry points now run on libgsv_b200")
    return old
