"""Rebind a live `gsv` (the reference package) onto the B200 path.

`gsv.cli` binds names at import (cli.py:23-25), so both the defining
modules and the CLI module are patched.  Results are converted
to the reference's own dataclasses, so callers see exactly the types they
expect; exceptions are the reference's classes (errors.py is shared).
"""

from __future__ import annotations


def install(verbose: bool = False) -> dict:
    import gsv  # noqa: F401  (the reference must be importable)
    import gsv.cli as gcli
    import gsv.codec as gcodec
    import gsv.container as gcont
    import gsv.gaussians as ggauss
    import gsv.motion as gmotion
    import gsv.pipeline as gpipe
    import gsv.quantize as gquant
    import gsv.render as grender

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

    patches = {
        (gpipe, "decode_video"): decode_video, (gcli, "decode_video"): decode_video,
        (gcont, "read_layers"): read_layers, (gpipe, "read_layers"): read_layers,
        (gcodec, "decode_planes"): decode_planes, (gcont, "decode_planes"): decode_planes,
        (grender, "render_set"): render_set, (gcli, "render_set"): render_set,
        (grender, "render_progressive"): render_progressive,
        (gmotion, "reconstruct_frame"): reconstruct_frame,
        (grender, "reconstruct_frame"): reconstruct_frame,
    }
    old = {}
    for (mod, name), fn in patches.items():
        if hasattr(mod, name):
            old[(mod.__name__, name)] = getattr(mod, name)
            setattr(mod, name, fn)
    for name in ("decode_video", "read_layers", "decode_planes", "render_set",
                 "render_progressive", "reconstruct_frame"):
        if hasattr(gsv, name):
            setattr(gsv, name, locals()[name])
    if verbose:
        print(f"gsv: {len(old)} entry points now run on libgsv_b200")
    return old
