"""Dev probe: what bounds the config-2 e2e step (render_sequence from pinned
host bytes to pinned u8 frames)?  Times, per 300-frame step (3 reps after a
warm-up):
  seq      render_sequence (H2D + open + render + D2H, the bench's e2e)
  rend     render_batch(device fp32 outs) on an open video (GPU only)
  rend_d2h render_batch(host_u8) on an open video (render + D2H)
  rend_h2d render_batch(device outs) + the container's H2D on a side stream
  d2h      300 x 6.2 MB device -> pinned copies alone (8 streams)
  h2d      the container's H2D alone"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
import paper_2509_17513_b200 as g
from paper_2509_17513_b200 import _lib


class A:
    gaussians, layers, frames, group, width, height = 300_000, 6, 300, 30, 1920, 1080


blobs, _ = bench.make_inputs(A, 1002)
data = blobs[0]
info = g.read_structure(data)
cs = _lib.camera_struct(bench.camera(A))
sess = g.Session(0)
hsrc = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
dcont = torch.empty(len(data), dtype=torch.uint8, device="cuda")
pinned = torch.empty((300, 1080, 1920, 3), dtype=torch.uint8).pin_memory()
dframe = torch.empty((1080, 1920, 3), dtype=torch.uint8, device="cuda")
outs = [torch.empty((1080, 1920, 3), dtype=torch.float32, device="cuda") for _ in range(300)]
res = torch.empty(len(data) + 64, dtype=torch.uint8, device="cuda")
res[:len(data)].copy_(hsrc)
v = g.DeviceVideo(data, 6, session=sess, resident=res, info=info, group_list=list(range(len(info.groups))))
side = torch.cuda.Stream()
cstreams = [torch.cuda.Stream() for _ in range(8)]
frames = list(range(300))


def seq():
    g.render_sequence(hsrc, cs, up_to_layer=6, out=pinned, session=sess, info=info)


def rend():
    v.render_batch(frames, cs, outs=outs, verify=False)
    sess.sync()


def rend_d2h():
    v.render_batch(frames, cs, host_u8=[pinned[i] for i in frames], verify=False)
    sess.sync()


def rend_h2d():
    with torch.cuda.stream(side):
        dcont.copy_(hsrc, non_blocking=True)
    v.render_batch(frames, cs, outs=outs, verify=False)
    sess.sync()
    side.synchronize()


def d2h():
    for i in frames:
        with torch.cuda.stream(cstreams[i % 8]):
            pinned[i].copy_(dframe, non_blocking=True)
    torch.cuda.synchronize()


def h2d():
    dcont.copy_(hsrc, non_blocking=True)
    torch.cuda.synchronize()


import ctypes
L = _lib.load()
L.gsv_dev_copy_h2d_stream.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int]


def h2dk(blocks=148):
    L.gsv_dev_copy_h2d_stream(dcont.data_ptr(), hsrc.data_ptr(), len(data) // 16 * 16, side.cuda_stream, blocks)
    side.synchronize()


def h2dk32():
    h2dk(32)


def rend_h2dk():
    L.gsv_dev_copy_h2d_stream(dcont.data_ptr(), hsrc.data_ptr(), len(data) // 16 * 16, side.cuda_stream, 32)
    v.render_batch(frames, cs, outs=outs, verify=False)
    sess.sync()
    side.synchronize()


sess2 = g.Session(0)
pinned2 = torch.empty((300, 1080, 1920, 3), dtype=torch.uint8).pin_memory()
import threading


def seq_b():
    g.render_sequence(hsrc, cs, up_to_layer=6, out=pinned2, session=sess2, info=info)


def seq2():
    """two sequences in flight (own session and output each): one step's
    upload head and read-back tail overlap the other's renders; counts as 2
    steps (reported per step)"""
    t = threading.Thread(target=lambda: (torch.cuda.set_device(0), seq_b()))
    t.start()
    seq()
    t.join()


only = sys.argv[1:]
for name, fn in (("seq", seq), ("seq2", seq2), ("seq", seq), ("seq2", seq2), ("rend", rend), ("rend_d2h", rend_d2h), ("rend_h2d", rend_h2d), ("d2h", d2h),
                 ("h2d", h2d), ("h2dk", h2dk), ("h2dk32", h2dk32), ("rend_h2dk", rend_h2dk), ("seq", seq)):
    if only and name not in only:
        continue
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    per = 6 if name == "seq2" else 3
    print(f"{name:9s} {(time.perf_counter() - t0) / per * 1e3:8.2f} ms/step", flush=True)
