"""ctypes binding of libgsv_b200.so (include/gsv_b200.h).

This is the reference-side binding a maintainer of `gsv` would add: the
reference is pure Python, so its FFI for the decode/render path is ctypes.
The library is built in-tree (paper_2509_17513_b200/lib/) by
``paper_2509_17513_b200.build``; there is no fallback: a missing library or
a missing CUDA device raises immediately.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import CodecError, FormatError, GsvError, InvalidInputError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libgsv_b200.so"

GSV_OK, GSV_E_INVALID_INPUT, GSV_E_FORMAT, GSV_E_CODEC, GSV_E_CUDA, GSV_E_NOMEM = range(6)


class GsvCudaError(GsvError, RuntimeError):
    """CUDA runtime failure inside libgsv_b200 (no reference counterpart)."""


class Camera_t(ctypes.Structure):
    _fields_ = [("rotation", ctypes.c_double * 9), ("translation", ctypes.c_double * 3),
                ("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("near_plane", ctypes.c_double),
                ("background", ctypes.c_double * 3), ("width", ctypes.c_int32),
                ("height", ctypes.c_int32)]


class Info_t(ctypes.Structure):
    _fields_ = [("version", ctypes.c_int32), ("layer_count", ctypes.c_int32),
                ("sh_degree", ctypes.c_int32), ("group_count", ctypes.c_int32),
                ("fps_num", ctypes.c_int32), ("fps_den", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("bounds", ctypes.c_float * 6),
                ("header_bytes", ctypes.c_uint64)]


class GroupInfo_t(ctypes.Structure):
    _fields_ = [("start_frame", ctypes.c_uint32), ("frame_count", ctypes.c_uint32),
                ("position_bits", ctypes.c_uint32), ("layer_counts", ctypes.c_uint32 * 64),
                ("channel_counts", ctypes.c_uint32 * 64)]


class EntryInfo_t(ctypes.Structure):
    _fields_ = [("attribute", ctypes.c_int32), ("component", ctypes.c_int32),
                ("bits", ctypes.c_int32), ("offset", ctypes.c_uint64), ("size", ctypes.c_uint64),
                ("range_min", ctypes.c_float), ("range_max", ctypes.c_float)]


class RenderStats_t(ctypes.Structure):
    _fields_ = [("n_splats", ctypes.c_int64), ("n_visible", ctypes.c_int64),
                ("n_keys", ctypes.c_int64), ("tiles_x", ctypes.c_int32), ("tiles_y", ctypes.c_int32),
                ("n_keys_emitted", ctypes.c_int64)]


class QuantChannel_t(ctypes.Structure):
    _fields_ = [("values", ctypes.c_void_p), ("planes", ctypes.c_void_p), ("frame_stride", ctypes.c_uint64),
                ("frames", ctypes.c_uint32), ("n", ctypes.c_uint32), ("width", ctypes.c_uint32),
                ("height", ctypes.c_uint32), ("bits", ctypes.c_uint32), ("range_min", ctypes.c_float),
                ("range_max", ctypes.c_float)]


class EncodeRun_t(ctypes.Structure):
    _fields_ = [("samples", ctypes.c_void_p), ("body", ctypes.c_void_p), ("count", ctypes.c_uint32),
                ("width", ctypes.c_uint32), ("height", ctypes.c_uint32), ("bits", ctypes.c_uint32),
                ("body_len", ctypes.c_uint64), ("checksum", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_SZ = ctypes.c_size_t

_SIGS = {
    "gsv_last_error": (ctypes.c_char_p, []),
    "gsv_last_error_kind": (_I, []),
    "gsv_abi_version": (_I, []),
    "gsv_session_create": (_I, [_I, ctypes.c_size_t, ctypes.POINTER(_P)]),
    "gsv_session_destroy": (None, [_P]),
    "gsv_session_sync": (_I, [_P]),
    "gsv_session_check_capacity": (_I, [_P]),
    "gsv_read_info": (_I, [_P, _SZ, ctypes.POINTER(Info_t)]),
    "gsv_read_group": (_I, [_P, _SZ, _I, ctypes.POINTER(GroupInfo_t)]),
    "gsv_read_directory": (_I, [_P, _SZ, _P, _SZ, _P, _SZ, ctypes.POINTER(_SZ)]),
    "gsv_read_entry": (_I, [_P, _SZ, _I, _I, _I, ctypes.POINTER(EntryInfo_t)]),
    "gsv_video_open": (_I, [_P, _P, _SZ, _I, ctypes.POINTER(_P)]),
    "gsv_video_open_groups": (_I, [_P, _P, _SZ, _I, _I, _I, ctypes.POINTER(_P)]),
    "gsv_video_open_resident": (_I, [_P, _P, _SZ, _P, _I, ctypes.POINTER(_P)]),
    "gsv_video_close": (None, [_P]),
    "gsv_video_open_group_list": (_I, [_P, _P, _SZ, _P, _I, _P, _I, _P]),
    "gsv_video_project_debug": (_I, [_P, _I, ctypes.POINTER(Camera_t), _P, _P, _P, _P,
                                     ctypes.POINTER(_I64)]),
    "gsv_video_frame_count": (_I, [_P]),
    "gsv_video_decoded_layers": (_I, [_P]),
    "gsv_video_group_of": (_I, [_P, _I]),
    "gsv_video_group_splats": (_I64, [_P, _I]),
    "gsv_video_frame_values": (_I, [_P, _I, _P, _P, _P, _P, _P]),
    "gsv_video_frame_codes": (_I, [_P, _I, _P]),
    "gsv_video_render": (_I, [_P, _I, ctypes.POINTER(Camera_t), _P, _P, _P]),
    "gsv_video_render_batch": (_I, [_P, _P, _I, ctypes.POINTER(Camera_t), _P, _P, _P, _I, _I]),
    "gsv_render_sequence_host": (_I, [_P, _P, _SZ, _I, _P, _I, ctypes.POINTER(Camera_t), _P, _I,
                                      ctypes.POINTER(_I64)]),
    "gsv_render_sequence": (_I, [_P, _P, _SZ, _P, _I, _P, _I, _P, _P, ctypes.POINTER(Camera_t), _P, _P, _P,
                                 _I, ctypes.POINTER(_I64)]),
    "gsv_render_soa": (_I, [_P, _I64, _I, _P, _P, _P, _P, _P, ctypes.POINTER(Camera_t), _P, _P,
                            _P]),
    "gsv_render_splats2d": (_I, [_P, _I64, _P, _P, _P, _P, _P, ctypes.POINTER(Camera_t), _P, _P, _P]),
    "gsv_sqdiff": (_I, [_P, _P, _P, _I64, _I, ctypes.POINTER(ctypes.c_double)]),
    "gsv_ssim": (_I, [_P, _P, _P, _I, _I, _I, ctypes.POINTER(ctypes.c_double)]),
    "gsv_fold_deltas": (_I, [_P, _I64, _I, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P]),
    "gsv_project_debug": (_I, [_P, _I64, _I, _P, _P, _P, _P, _P, ctypes.POINTER(Camera_t), _P, _P,
                               _P, _P, ctypes.POINTER(_I64)]),
    "gsv_decode_payload_host": (_I, [_P, _P, _SZ, _P, _SZ, _P]),
    "gsv_encode_reference_body": (_I64, [_P, _I, _I, _I, _I, _P, _SZ]),
    "gsv_quantize_channels": (_I, [_P, _P, _I]),
    "gsv_encode_body_capacity": (ctypes.c_uint64, [ctypes.c_uint32] * 4),
    "gsv_encode_runs": (_I, [_P, _P, _I]),
    "gsv_crc32": (ctypes.c_uint32, [_P, _SZ]),
    "gsv_kernel_launches": (ctypes.c_longlong, []),
    "gsv_profile_enable": (_I, [_I]),
    "gsv_profile_read": (_I, [_P, _P, _I]),
}

_lib = None


def load():
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        if os.environ.get("GSV_B200_AUTOBUILD", "1") == "1":
            from . import build as _build
            _build.build()
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing; run `python -m paper_2509_17513_b200.build`")
    L = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == GSV_OK:
        return
    msg = load().gsv_last_error().decode(errors="replace")
    if rc == GSV_E_INVALID_INPUT:
        raise InvalidInputError(msg)
    if rc == GSV_E_FORMAT:
        raise FormatError(msg)
    if rc == GSV_E_CODEC:
        raise CodecError(msg)
    if rc == GSV_E_NOMEM:
        raise MemoryError(msg)
    raise GsvCudaError(msg)


STAGES = ("project", "depth_sort", "key_emit", "tile_sort", "tile_ranges", "composite",
          "range_decode", "crc")


def profile_enable(on: bool = True) -> None:
    load().gsv_profile_enable(1 if on else 0)


def profile_read() -> dict:
    import numpy as np
    ms = np.zeros(len(STAGES), np.float64)
    n = np.zeros(len(STAGES), np.int64)
    load().gsv_profile_read(ms.ctypes.data, n.ctypes.data, len(STAGES))
    return {s: {"ms": float(ms[i]), "intervals": int(n[i])} for i, s in enumerate(STAGES)}


def kernel_launches() -> int:
    return int(load().gsv_kernel_launches())


def camera_struct(cam) -> Camera_t:
    import numpy as np
    c = Camera_t()
    c.rotation[:] = [float(x) for x in np.asarray(cam.rotation, dtype=np.float64).ravel()]
    c.translation[:] = [float(x) for x in np.asarray(cam.translation, dtype=np.float64).ravel()]
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.near_plane = float(getattr(cam, "near", 0.01))
    c.background[:] = [float(x) for x in getattr(cam, "background", (0.0, 0.0, 0.0))]
    c.width, c.height = int(cam.width), int(cam.height)
    return c
