"""Dev diagnostic: host timeline of the per-group pipelined e2e loop."""
import sys, time, threading
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
import paper_2509_17513_b200 as gsvb
from paper_2509_17513_b200 import _lib

class A:
    gaussians, layers, frames, group, width, height, k, streams = 300_000, 6, 300, 30, 1920, 1080, 6, 8
a = A()
blobs, _ = bench.make_inputs(a, 1002)
blob = blobs[0]
cs = _lib.camera_struct(bench.camera(a))
info = gsvb.read_structure(blob)
host = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
pinned = torch.empty((a.frames, a.height, a.width, 3), dtype=torch.uint8).pin_memory()
import os
NW = int(os.environ.get('NW', '4'))
sessions = [gsvb.Session(0) for _ in range(NW)]
log = []
T0 = [0.0]
def ev(*x): log.append((time.perf_counter() - T0[0], threading.get_ident() % 100) + x)
first = [threading.Event() for _ in range(NW)]
def worker(w, verify):
    torch.cuda.set_device(0)
    if w >= 1: first[w - 1].wait()
    for gi in range(w, len(info.groups), NW):
        g = info.groups[gi]
        ev("open", gi)
        v = gsvb.DeviceVideo(host, a.k, session=sessions[w], groups=(gi, gi + 1), info=info)
        first[w].set()
        ev("opened", gi)
        hf = [pinned[gi * 30 + i] for i in range(g.frame_count)]
        v.render_batch(list(range(g.frame_count)), cs, host_u8=hf, streams=a.streams, verify=verify)
        ev("enqueued", gi)
        v.close()
        ev("closed", gi)
from concurrent.futures import ThreadPoolExecutor
pool = ThreadPoolExecutor(NW)
for it in range(3):
    log.clear(); [e.clear() for e in first]; torch.cuda.synchronize(); T0[0] = time.perf_counter()
    for f in [pool.submit(worker, w, it == 0) for w in range(NW)]: f.result()
    torch.cuda.synchronize()
    tot = time.perf_counter() - T0[0]
print(f"step {tot*1e3:.1f} ms")
# render alone (container resident) for reference
res = torch.empty(len(blob) + 64, dtype=torch.uint8, device="cuda"); res[:len(blob)].copy_(host[:len(blob)].cuda())
for it in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    v = gsvb.DeviceVideo(blob, a.k, session=sessions[0], resident=res, info=info)
    v.render_batch(list(range(300)), cs, host_u8=[pinned[i] for i in range(300)], streams=8, verify=False); v.close()
    torch.cuda.synchronize(); print(f"resident + D2H {1e3*(time.perf_counter()-t):.1f} ms")
    torch.cuda.synchronize(); t = time.perf_counter()
    v = gsvb.DeviceVideo(blob, a.k, session=sessions[0], resident=res, info=info)
    outs = [torch.empty((1080,1920,3), dtype=torch.uint8, device='cuda') for _ in range(8)]
    v.render_batch(list(range(300)), cs, outs_u8=[outs[i % 8] for i in range(300)], streams=8, verify=False); v.close()
    torch.cuda.synchronize(); print(f"resident, device u8 {1e3*(time.perf_counter()-t):.1f} ms")
for e in log: print(f"{e[0]*1e3:8.2f} ms thr{e[1]:02d} {e[2]:9s} g{e[3]}")
