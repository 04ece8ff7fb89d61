"""Range-decoder micro-benchmark (dev tool): decode single codec-1 runs of the
config-2 scene (30-frame group, 224x224 planes) on the GPU, check them
bit-exact against the oracle, time each decoder variant (GSV_RC_VARIANT).

usage: rc_bench.py [--planes K] [variants...]   (K: truncate runs to K planes)"""
import ctypes
import os
import struct
import sys
import time
import zlib
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import bench
import paper_2509_17513_b200 as g
from oracle import oracle as O
from paper_2509_17513_b200 import _lib


class A:
    gaussians, layers, frames, group, width, height = 300_000, 6, 30, 30, 1920, 1080


def truncate(blob, k):
    """Rebuild a flag-0 codec-1 payload keeping its first k planes."""
    codec, bits, w, h, count, _, length = struct.unpack_from("<BBHHHHI", blob, 0)
    body = blob[14:14 + length]
    assert codec == 1 and body[0] == 0
    modes = body[1:1 + count]
    pos, blocks = 1 + count, []
    for f in range(count):
        if modes[f] == 1:
            n = w * h * bits // 8
        else:
            n = 4 + struct.unpack_from("<I", body, pos)[0]
        blocks.append(body[pos:pos + n])
        pos += n
    nb = bytes([0]) + bytes(modes[:k]) + b"".join(blocks[:k])
    _, planes = O.decode_payload(blob)
    le = {8: "<u1", 16: "<u2", 32: "<u4"}[bits]
    crc = zlib.crc32(planes[:k].astype(le).tobytes()) & 0xFFFFFFFF
    return struct.pack("<BBHHHHI", codec, bits, w, h, k, 0, len(nb)) + nb + struct.pack("<I", crc)


args = sys.argv[1:]
k = None
if args and args[0] == "--planes":
    k = int(args[1])
    args = args[2:]
variants = [int(v) for v in (args or ["1", "2"])]
blobs, _ = bench.make_inputs(A, 1002)
data = blobs[1]
info = g.read_structure(data)
picks = {}
for e in info.groups[0].channels[0]:
    blob = data[e.offset:e.offset + e.size]
    picks.setdefault(blob[1], blob)
slow_fn = _lib.load().gsv_dev_rc_slow_bytes
slow_fn.restype = ctypes.c_ulonglong
for bits, blob in sorted(picks.items()):
    if k:
        blob = truncate(blob, k)
    _, ref = O.decode_payload(blob)
    for v in variants:
        os.environ["GSV_RC_VARIANT"] = str(v)
        g.decode_planes(g.CodedPayload.from_bytes(blob)[0])  # warm
        slow_fn(1)
        t0 = time.perf_counter()
        planes = g.decode_planes(g.CodedPayload.from_bytes(blob)[0])
        dt = time.perf_counter() - t0
        got = np.stack([p.samples for p in planes])
        ok = np.array_equal(got.astype(np.int64).ravel(), ref.astype(np.int64).ravel())
        dec = (got.shape[0] - 1) * got.shape[1] * got.shape[2] * bits  # plane 0 is RAW here
        print(f"bits={bits} variant={v} ok={ok} {dt * 1e3:.1f} ms  {dt / dec * 1e9 * 1.965:.1f} cycles/decision"
              f"  slow bytes {slow_fn(1)}", flush=True)
