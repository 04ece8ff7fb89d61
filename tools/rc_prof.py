"""Range-decoder in-situ profile (dev tool): open the config-2 codec-1
container (10 groups x 138 runs, resident in HBM) and report, per channel,
the decode cycles of its runs (clock64 from the first plane to the last,
recorded by the kernel when gsv_dev_rc_profile is set) and cycles per sample,
plus the open's CUDA-event time, for each setting given as ENV=VAL,... .

usage: rc_prof.py [setting ...]   e.g.  rc_prof.py GSV_RC_ORDER=0 GSV_RC_ORDER=1 GSV_RC_RPW=8"""
import ctypes
import os
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
import paper_2509_17513_b200 as g
from paper_2509_17513_b200 import _lib


class A:
    gaussians, layers, frames, group, width, height = 300_000, 6, 300, 30, 1920, 1080


settings = sys.argv[1:] or [""]
blobs, _ = bench.make_inputs(A, 1002)
data = blobs[1]
res = torch.empty(len(data) + 64, dtype=torch.uint8, device="cuda")
res[:len(data)].copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
info = g.read_structure(data)
chan_of = []
for gd in info.groups:
    for l in range(info.layer_count):
        for e in gd.channels[l]:
            chan_of.append((e.channel.attribute, e.channel.component, gd.frame_count))
L = _lib.load()
L.gsv_dev_rc_profile.argtypes = [ctypes.c_void_p]
L.gsv_dev_rc_slow_bytes.restype = ctypes.c_ulonglong
prof = torch.zeros(2 * len(chan_of), dtype=torch.int64, device="cuda")
sess = g.Session()
base_env = dict(os.environ)
ref_codes = None
for st in settings:
    os.environ.clear()
    os.environ.update(base_env)
    for kv in filter(None, st.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    times = []
    L.gsv_dev_rc_slow_bytes(1)
    for rep in range(2):
        prof.zero_()
        L.gsv_dev_rc_profile(ctypes.c_void_p(prof.data_ptr()))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sess.stream)
        try:
            vid = g.DeviceVideo(data, 6, session=sess, resident=res, info=info)
        except g.CodecError:  # GSV_RC_SKIP probes leave runs undecoded (by design)
            torch.cuda.synchronize()
            times.append(float("nan"))
            same = None
            continue
        e1.record(sess.stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        if rep == 0:
            codes = [vid.frame_codes(t).cpu() for t in (1, 29, 150, 299)]
            if ref_codes is None:
                ref_codes = codes
            same = all(torch.equal(a, b) for a, b in zip(ref_codes, codes))
        vid.close()
    L.gsv_dev_rc_profile(ctypes.c_void_p(0))
    p = prof.view(-1, 2).cpu().numpy()
    per = defaultdict(list)
    for rid, cyc in p:
        if cyc > 0:
            a, c, fc = chan_of[rid]
            per[(a, c)].append(cyc)
    hw = 224 * 224
    slow = L.gsv_dev_rc_slow_bytes(1)
    print(f"== [{st or 'default'}] open {min(times):.1f} ms  codes == first setting: {same}  "
          f"careful-path bytes (lane calls, 2 opens) {slow}")
    rows = sorted(per.items(), key=lambda kv: -max(kv[1]))
    for (a, c), cyc in rows[:8]:
        print(f"   {a}[{c}]: runs {len(cyc)}  max {max(cyc) / 1e6:.1f} Mcyc  mean {sum(cyc) / len(cyc) / 1e6:.1f} Mcyc"
              f"  = {max(cyc) / (30 * hw):.0f} cyc/sample (max)")
    allc = [x for v in per.values() for x in v]
    print(f"   all: max {max(allc) / 1e6:.1f} Mcyc  ({max(allc) / 1.965e6:.0f} ms at 1965 MHz)", flush=True)
