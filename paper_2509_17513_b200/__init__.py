"""B200-native decode-and-render path of 4DGCPro's `gsv` package.

Drop-in for the reference's decode/render entry points (see api.py); the
compute runs in hand-written sm_100a CUDA kernels in lib/libgsv_b200.so,
bound through the C ABI in include/gsv_b200.h.
"""

from .errors import CodecError, FormatError, GsvError, InvalidInputError, StreamError
from .types import (Camera, ChannelEntry, ChannelId, CodedPayload, ContainerInfo, DecodedGroup,
                    DecodedVideo, FrameDelta, GaussianSet, GroupDirectory, Image, LayeredFrame,
                    Plane, ResidualDelta, RigidDelta, Splat2D, load_camera, sh_coeff_count)

__version__ = "0.1.0"

_API = ("DeviceVideo", "Session", "analyze_rd", "d_ssim", "decode_planes", "decode_video",
        "default_session", "load_raw_floats", "project_debug", "psnr", "read_container_info", "read_layers",
        "read_structure", "reconstruct_frame", "reconstruct_frame_tensors", "render",
        "render_progressive", "render_sequence", "render_set", "render_soa_tensors", "ssim", "write_ppm",
        "write_raw_floats")


def __getattr__(name):  # lazy: importing torch is only needed for the GPU API
    if name in _API:
        from . import api
        return getattr(api, name)
    if name == "install":
        from .install import install
        return install
    raise AttributeError(name)


__all__ = ["CodecError", "FormatError", "GsvError", "InvalidInputError", "StreamError", "Camera",
           "ChannelEntry", "ChannelId", "CodedPayload", "ContainerInfo", "DecodedGroup",
           "DecodedVideo", "FrameDelta", "GaussianSet", "GroupDirectory", "Image", "LayeredFrame",
           "Plane", "ResidualDelta", "RigidDelta", "Splat2D", "load_camera", "sh_coeff_count", *_API]
