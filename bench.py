"""Benchmark: decoded+rendered 1080p frames/sec (BASELINE config 2).

Workload: a synthetic 300k-Gaussian, 6-layer, 300-frame sequence (10 motion
groups, SH degree 1; SURVEY 8(d) recipe, seed 1002 + rank) encoded with the
reference's bitstream; camera looking_at(eye=(0,0,-2.5)), 60 deg, 1920x1080.
One step = decode layers 1..k of the whole container (range decode + CRC of
every run, as decode_video does) and render every frame at 1080p.  The
headline is k = 6 with codec 0 (raw planes: decode = CRC-32 validation of
every run + zero-copy planes); codec 1 (the reference's default adaptive
range coder, strictly serial within a run) and the per-layer sweep k = 1..6
for both codecs are reported alongside.  Frames render frame-parallel on
--streams CUDA streams.

value: container bytes already resident in HBM (gsv_video_open_resident),
       CUDA events on the session stream, max over ranks.
e2e:   the public API with HOST buffers: per group, DeviceVideo(host bytes,
       groups=(g, g+1)) (gsv_video_open_groups: H2D of the layer-prefix bytes,
       decode, CRC) + render_batch with a D2H of every frame as u8 RGB into
       pinned memory, two sessions in turn so uploads overlap rendering; host
       wall clock around whole steps.
Multi-GPU: one process per GPU, each rank decodes+renders its own sequence
(no data-path collective; weak scaling); a gloo/NCCL all_reduce(max) of the
times after the barrier.

--impl reference: times the CPU oracle (oracle/, the restatement of the
reference's decode_video + render_set; the reference package itself is
pure Python and cannot travel to the GPU box) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decoded+rendered 1080p frames/sec (layers L1-L6; ms/frame; HBM roofline %)"
CACHE = Path(os.environ.get("GSV_BENCH_CACHE", "/tmp/gsv_bench_cache"))


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--gaussians", type=int, default=300_000)
    p.add_argument("--layers", type=int, default=6)
    p.add_argument("--frames", type=int, default=300)
    p.add_argument("--group", type=int, default=30)
    p.add_argument("--width", type=int, default=1920)
    p.add_argument("--height", type=int, default=1080)
    p.add_argument("--k", type=int, default=6, help="layer prefix of the headline")
    p.add_argument("--codec", type=int, default=0, choices=[0, 1])
    p.add_argument("--no-sweep", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-sample-frames", type=int, default=2)
    p.add_argument("--streams", type=int, default=8)
    p.add_argument("--short-groups", action="store_true",
                   help="also time both codecs with config 3's grouping (a burst every 2 frames: "
                        "150 motion groups) at config 2's size")
    p.add_argument("--multiview", action="store_true",
                   help="also run BASELINE config 4's shape on this GPU: 500k Gaussians, 16 ring "
                        "cameras, k = 1..6 (60 frames)")
    return p.parse_args()


# ---------------------------------------------------------------------------
def make_inputs(a, seed):
    """Container bytes for both codecs (cached on local disk by recipe)."""
    from paper_2509_17513_b200.encode import EncodeConfig, encode_stream
    from paper_2509_17513_b200.synth import benchmark_spec, iter_frames
    key = hashlib.sha256(json.dumps([a.gaussians, a.layers, a.frames, a.group, seed, 3]).encode()
                         ).hexdigest()[:16]
    paths = {c: CACHE / f"{key}_c{c}.gsv" for c in (0, 1)}
    if all(p.exists() for p in paths.values()):
        return {c: p.read_bytes() for c, p in paths.items()}, key
    spec = benchmark_spec(a.gaussians, a.frames, a.group)
    cfg = EncodeConfig(layer_count=a.layers, prune_fraction=0.0, motion_threshold=0.0025)
    t0 = time.time()
    import torch
    # the GPU encoder when a device is present (byte-identical to the host coder)
    blobs = encode_stream(lambda: iter_frames(spec, seed), cfg, codecs=(0, 1),
                          positions_source=lambda: iter_frames(spec, seed, positions_only=True),
                          device=True if torch.cuda.is_available() else None)
    print(f"[bench] encoded {a.frames} frames x {a.gaussians} in {time.time() - t0:.1f}s",
          file=sys.stderr, flush=True)
    CACHE.mkdir(parents=True, exist_ok=True)
    for c, p in paths.items():
        tmp = p.with_suffix(".tmp")
        tmp.write_bytes(blobs[c])
        os.replace(tmp, p)
    return blobs, key


def ring_cameras(a, views=16):
    """looking_at cameras on a radius-2.5 ring, 22.5 deg
    steps, elevation +-10 deg alternating, 60 deg fov."""
    import math
    from paper_2509_17513_b200.types import Camera
    cams = []
    for v in range(views):
        az = math.radians(22.5 * v)
        el = math.radians(10.0 if v % 2 == 0 else -10.0)
        eye = (2.5 * math.cos(el) * math.sin(az), 2.5 * math.sin(el), -2.5 * math.cos(el) * math.cos(az))
        cams.append(Camera.looking_at(eye=eye, target=(0.0, 0.0, 0.0), fov_deg=60.0,
                                      width=a.width, height=a.height, near=0.01))
    return cams


def run_multiview(a, sess, dev):
    """Config 4 on one GPU: per layer prefix k, decode the container once
    (resident in HBM) and render every frame from 16 cameras.  Metric:
    rendered 1080p images/s (decode included)."""
    import copy

    import torch

    import paper_2509_17513_b200 as gsvb
    from paper_2509_17513_b200 import _lib
    m = copy.copy(a)
    m.gaussians, m.frames, m.group = 500_000, 60, 30
    blobs, _ = make_inputs(m, 1004)
    data = blobs[0]
    dinfo = gsvb.read_structure(data)  # the directory, parsed once per container
    res = torch.empty(len(data) + 64, dtype=torch.uint8, device="cuda")
    res[:len(data)].copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
    cams = [_lib.camera_struct(c) for c in ring_cameras(m)]
    outs = [torch.empty((m.height, m.width, 3), dtype=torch.float32, device="cuda") for _ in range(m.frames)]
    frames = list(range(m.frames))
    out = {}
    for k in range(1, m.layers + 1):
        def step(verify=False):
            v = gsvb.DeviceVideo(data, k, session=sess, resident=res, info=dinfo)
            for c in cams:
                v.render_batch(frames, c, outs=outs, streams=a.streams, verify=verify)
            v.close()
        step(verify=True)
        s = sess.stream
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        step()
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        imgs = m.frames * len(cams)
        out[str(k)] = {"images_per_s": round(imgs / (ms / 1e3), 1), "ms": round(ms, 2)}
    return {"workload": "config4 shape on 1 GPU: 500k Gaussians, 6 layers, 60 frames (2 groups), "
                        "16 ring cameras, 1080p, codec 0, container resident",
            "per_layer": out}


def run_short_groups(a, sess):
    """Config 3's adaptive grouping (2-frame motion groups, bursts every 2
    frames) at config 2's size: the range decoder's serial chain per run is
    1 plane long instead of 29, and 150 groups decode in parallel.  Same step
    as the headline (open + decode + CRC + render of all frames, container
    resident), both codecs, k = 6."""
    import copy

    import torch

    import paper_2509_17513_b200 as gsvb
    from paper_2509_17513_b200 import _lib
    m = copy.copy(a)
    m.group = 2
    blobs, _ = make_inputs(m, 1003)
    cs = _lib.camera_struct(camera(m))
    outs = [torch.empty((m.height, m.width, 3), dtype=torch.float32, device="cuda") for _ in range(m.frames)]
    res = {}
    for codec in (0, 1):
        data = blobs[codec]
        dinfo = gsvb.read_structure(data)  # the directory, parsed once per container
        dev = torch.empty(len(data) + 64, dtype=torch.uint8, device="cuda")
        dev[:len(data)].copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))

        def step(verify=False):
            v = gsvb.DeviceVideo(data, m.layers, session=sess, resident=dev, info=dinfo)
            v.render_batch(list(range(m.frames)), cs, outs=outs, streams=a.streams, verify=verify)
            v.close()
        step(verify=True)
        s = sess.stream
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(2):
            step()
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 2
        res[f"codec{codec}"] = {"fps": round(m.frames / (ms / 1e3), 1), "ms_per_step": round(ms, 2),
                                "container_mb": round(len(data) / 1e6, 1)}
    return {"workload": "config3 grouping at config2 size: 300k Gaussians, 6 layers, 300 frames in "
                        "150 two-frame motion groups, 1080p, k = 6, container resident", **res}


def camera(a):
    from paper_2509_17513_b200.types import Camera
    return Camera.looking_at(eye=(0.0, 0.0, -2.5), target=(0.0, 0.0, 0.0), fov_deg=60.0,
                             width=a.width, height=a.height, near=0.01)


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower() in ("active", "0x1", "1")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
def run_b200(a, rank, world, dist):
    import numpy as np
    import torch

    import paper_2509_17513_b200 as gsvb
    from paper_2509_17513_b200 import _lib

    dev = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    blobs, key = make_inputs(a, 1002 + rank)
    cam = camera(a)
    cs = _lib.camera_struct(cam)
    sess = gsvb.Session(dev)
    s = sess.stream
    resident = {}
    infos = {c: gsvb.read_structure(b) for c, b in blobs.items()}  # directories, parsed once
    for c, b in blobs.items():
        t = torch.empty(len(b) + 64, dtype=torch.uint8, device="cuda")
        t[:len(b)].copy_(torch.frombuffer(bytearray(b), dtype=torch.uint8))
        resident[c] = t
    torch.cuda.synchronize()
    # every decoded frame keeps its own fp32 image in HBM (7.5 GB at 300 x 1080p)
    outs = [torch.empty((a.height, a.width, 3), dtype=torch.float32, device="cuda")
            for _ in range(a.frames)]
    frames = list(range(a.frames))

    def step_resident(codec, k, verify=False, streams=None):
        v = gsvb.DeviceVideo(blobs[codec], k, session=sess, resident=resident[codec], info=infos[codec])
        v.render_batch(frames, cs, outs=outs, streams=streams or a.streams, verify=verify)
        return v

    # size the key buffers (stats path + one checked batch per codec)
    for codec in (0, 1):
        v = gsvb.DeviceVideo(blobs[codec], a.layers, session=sess, resident=resident[codec],
                             info=infos[codec])
        _, st0 = v.render(0, cam, stats=True)
        v.close()
        step_resident(codec, a.layers, verify=True).close()

    host_ms = [0.0]
    local_ms = [0.0]

    def timed(codec, k, steps, warmup, e2e=False):
        pinned = None
        if e2e:
            pinned = torch.empty((a.frames, a.height, a.width, 3), dtype=torch.uint8).pin_memory()
            host_frames = [pinned[t] for t in range(a.frames)]
            host = torch.frombuffer(bytearray(blobs[codec]), dtype=torch.uint8).pin_memory()

        def one(verify=False):
            if not e2e:
                return step_resident(codec, k, verify=verify)
            v = gsvb.DeviceVideo(host, k, session=sess, info=infos[codec])
            v.render_batch(frames, cs, host_u8=host_frames, streams=a.streams, verify=verify)
            return v

        for _ in range(warmup):  # the checked warm-up steps size the key buffers
            one(verify=True).close()
        s.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches0 = _lib.kernel_launches()
        t_host0 = time.perf_counter()
        e0.record(s)
        t_enq = 0.0
        for _ in range(steps):
            t1 = time.perf_counter()
            v = one()
            t_enq += time.perf_counter() - t1  # host time to open + enqueue the step
            v.close()
        e1.record(s)
        e1.synchronize()
        t_host = time.perf_counter() - t_host0
        launches = _lib.kernel_launches() - launches0
        _lib.check(sess.lib.gsv_session_check_capacity(sess.handle))
        ms = e0.elapsed_time(e1)
        # decode happens inside open(): its host-side part is inside the event
        # window because the events bracket every call on the same stream
        host_ms[0] = t_enq * 1e3 / steps
        ms = max(ms, t_host * 1e3)
        local_ms[0] = ms
        torch.cuda.synchronize()
        if dist:
            tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        nfr = steps * a.frames * world
        return nfr / (ms / 1e3), ms / steps, launches

    with Clocks(dev) as clk:
        fps, ms_step, launches = timed(a.codec, a.k, a.steps, a.warmup)
    clocks = clk.summary()
    # per-rank metrics gathered to rank 0 over NCCL (after the timed region):
    # each rank's own step time and a checksum of its last rendered frame
    ranks = None
    if dist:
        mine = torch.tensor([float(rank), local_ms[0] / a.steps, float(outs[-1].double().sum())],
                            dtype=torch.float64, device="cuda")
        got = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(got, mine)
        ranks = [{"rank": int(x[0].item()), "ms_per_step": round(x[1].item(), 3),
                  "last_frame_sum": round(x[2].item(), 3)} for x in got]
    host_ms_step = host_ms[0]

    # stage profile of one step (separate pass: events perturb timing slightly)
    _lib.profile_enable(True)
    v = step_resident(a.codec, a.k, streams=1)
    s.synchronize()
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    v.close()

    sweep = {}
    if not a.no_sweep:
        for codec in (0, 1):
            sweep[f"codec{codec}"] = {}
            for k in range(1, a.layers + 1):
                f, m, _ = timed(codec, k, max(1, a.steps // 2), 1)
                sweep[f"codec{codec}"][str(k)] = {"fps": round(f, 1),
                                                  "ms_per_frame": round(1e3 / f * world, 4)}
    e2e = None
    if not a.no_e2e:
        f, m = timed_e2e_pipelined(a, gsvb, sess, blobs[a.codec], cs, max(1, a.steps // 2), 1, dist)
        info = gsvb.read_structure(blobs[a.codec])
        h2d = 0
        for g in info.groups:
            offs = [e.offset for l in range(a.k) for e in g.channels[l]]
            ends = [e.offset + e.size for l in range(a.k) for e in g.channels[l]]
            h2d += max(ends) - min(offs)
        e2e = {"value": round(f, 2), "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(a.frames * a.width * a.height * 3),
               "path": "per-group DeviceVideo(host, groups=(g, g+1)) + render_batch(host_u8), "
                       f"{os.environ.get('GSV_E2E_WORKERS', '3')} host threads / sessions",
               "whole_container_open_fps": round(timed_e2e_pipelined.whole_fps, 2),
               "pcie_floor_ms_per_step": "H2D 42 + D2H 34 concurrently 51 (tools/pcie_probe.py)"}

    multiview = run_multiview(a, sess, dev) if a.multiview else None
    short_groups = run_short_groups(a, sess) if a.short_groups else None

    # roofline of the dominant stage (CUDA events around its launches on the
    # launching stream, one single-stream step)
    stage_ms = {k: v["ms"] for k, v in prof.items()}
    dom = max(stage_ms, key=stage_ms.get)
    roof = roofline(a, blobs[a.codec], dom, prof, st0, a.evals_per_frame)
    frame_bytes = (len(blobs[a.codec]) / a.frames
                   + sum(stage_bytes(a, blobs[a.codec], k, st0) / a.frames
                         for k in ("project", "depth_sort", "key_emit", "tile_sort", "composite")))
    result = {
        "metric": METRIC, "value": round(fps, 2), "unit": "frames/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_step, 3),
        "ms_per_frame": round(ms_step / a.frames, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32",
        "data": "synthetic (SURVEY 8(d) recipe, reference bitstream, seed 1002+rank)",
        "config": {"workload": "config2: 300k Gaussians, 6 layers, 300 frames (10 groups), "
                               "1080p, single camera",
                   "gaussians": a.gaussians, "layers": a.layers, "frames": a.frames,
                   "groups": a.frames // a.group, "resolution": [a.width, a.height],
                   "k": a.k, "codec": a.codec, "parallelism": f"frame-sharded x{world}",
                   "l2": f"inputs larger than L2 ({len(blobs[a.codec]) / 1e6:.0f} MB container)"},
        "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
        "host_enqueue_ms_per_step": round(host_ms_step, 3),
        "roofline": roof, "stages_ms_per_frame": {k: round(v["ms"] / a.frames, 5)
                                                  for k, v in prof.items()},
        "render_stats": st0, "per_layer": sweep,
        **({"ranks": ranks} if ranks else {}),
        **({"multiview": multiview} if multiview else {}),
        **({"short_groups": short_groups} if short_groups else {}),
        # whole-frame HBM roofline: algorithmic bytes of one
        # decoded+rendered frame x fps against the HBM peak
        "frame_roofline": {"bytes_per_frame": int(frame_bytes),
                           "achieved_gbs": round(frame_bytes * fps / 1e9, 1),
                           "peak_gbs": peaks()[0], "frac": round(frame_bytes * fps / 1e9 / peaks()[0], 4)},
    }
    return result


def timed_e2e_pipelined(a, gsvb, sess, blob, cs, steps, warmup, dist):
    """e2e through the public API with HOST buffers: the container in pinned
    host memory, every frame read back as u8 RGB into pinned host memory.
    Groups are opened one at a time (DeviceVideo(..., groups=(g, g+1)):
    H2D of the group's layer-prefix bytes, decode, CRC) by GSV_E2E_WORKERS
    host threads, each with its own session, so uploads and validation of
    some groups overlap rendering and read-back of others.  Host wall clock
    around whole steps, device synchronised."""
    import torch
    info = gsvb.read_structure(blob)
    host = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
    pinned = torch.empty((a.frames, a.height, a.width, 3), dtype=torch.uint8).pin_memory()
    starts, acc = [], 0
    for g in info.groups:
        starts.append(acc)
        acc += g.frame_count
    nw = int(os.environ.get("GSV_E2E_WORKERS", "3"))
    sessions = [sess] + [gsvb.Session(sess.device) for _ in range(nw - 1)]
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max_workers=nw)

    import threading
    opened = [threading.Event() for _ in range(len(info.groups))]

    def worker(w, verify):
        # host thread w drives session w over groups w, w+nw, ... (the C ABI
        # releases the GIL); group g is opened only after group g-1 is open,
        # so the uploads go one at a time at full PCIe rate, in group order,
        # while the other threads render and read back
        torch.cuda.set_device(sess.device)
        for gi in range(w, len(info.groups), nw):
            g = info.groups[gi]
            if gi > 0:
                opened[gi - 1].wait()
            v = gsvb.DeviceVideo(host, a.k, session=sessions[w], groups=(gi, gi + 1), info=info)
            opened[gi].set()
            hf = [pinned[starts[gi] + i] for i in range(g.frame_count)]
            v.render_batch(list(range(g.frame_count)), cs, host_u8=hf, streams=a.streams, verify=verify)
            v.close()

    def one(verify=False):
        for e in opened:
            e.clear()
        for f in [pool.submit(worker, w, verify) for w in range(nw)]:
            f.result()

    for _ in range(warmup):
        one(verify=True)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    # the whole-container open (one gsv_video_open of all groups, then render)
    # for comparison
    v = gsvb.DeviceVideo(host, a.k, session=sess, info=info)
    v.render_batch(list(range(a.frames)), cs, host_u8=[pinned[t] for t in range(a.frames)],
                   streams=a.streams, verify=True)
    v.close()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(steps):
        v = gsvb.DeviceVideo(host, a.k, session=sess, info=info)
        v.render_batch(list(range(a.frames)), cs, host_u8=[pinned[t] for t in range(a.frames)],
                       streams=a.streams, verify=False)
        v.close()
    torch.cuda.synchronize()
    ms_whole = (time.perf_counter() - t1) * 1e3
    print(f"[bench] e2e per-group pipelined {ms / steps:.1f} ms/step, whole-container {ms_whole / steps:.1f} ms/step",
          file=sys.stderr, flush=True)
    world_ = dist.get_world_size() if dist else 1
    timed_e2e_pipelined.whole_fps = steps * a.frames * world_ / (ms_whole / 1e3)
    if dist:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    world = dist.get_world_size() if dist else 1
    return steps * a.frames * world / (ms / 1e3), ms / steps


def stage_bytes(a, blob, stage, st):
    """Algorithmic HBM bytes of one step for a stage:
    what the stage must move at minimum, per frame x frames."""
    n, nvis = st["n_splats"], st["n_visible"]
    k_emit = st["n_keys_emitted"]
    npx = a.width * a.height
    per_frame = {
        # codes in (26 B/splat at SH degree 1), depth key + index + 64-B record out
        "project": 26 * n + 12 * n + 64 * nvis,
        # 3 passes (24-bit key): read + write (4-B key, 4-B index)
        "depth_sort": 3 * 2 * 8 * n,
        # key emission: rank -> index, the record's rect (8 B), the (tile, index) keys out
        "key_emit": (4 + 8) * nvis + 8 * k_emit,
        # 2 passes over the emitted (tile, rank) keys
        "tile_sort": 2 * 2 * 8 * k_emit,
        "tile_ranges": 0,
        # per emitted key: splat index + 48 B of the record used; the fp32 image out
        "composite": (4 + 48) * k_emit + 12 * npx,
    }
    if stage in per_frame:
        return per_frame[stage] * a.frames
    return len(blob)  # decode stages: the container bytes read once per step


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md: MEASURED_PEAKS.json absent)"


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full capture summary (profiles/ncu_traffic.json)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(kernel)


KERNEL_OF = {"composite": "composite_strip_kernel", "project": "project_kernel",
             "depth_sort": "radix_onesweep", "tile_sort": "radix_onesweep",
             "key_emit": "round_emit_fused", "range_decode": "rc_decode_kernel", "crc": "crc_kernel"}
MUFU_EX2_PER_CLK_SM = 16          # B200 SFU rate (ex2.approx), per SM per clock
SMS, SM_MHZ_MAX = 148, 1965.0


def roofline(a, blob, stage, prof, st, evals_per_frame):
    peak, src = peaks()
    ms = prof[stage]["ms"]
    launches = int(prof[stage].get("intervals", 0))
    b = stage_bytes(a, blob, stage, st)
    achieved = b / (ms / 1e3) / 1e9 if ms > 0 else 0.0
    tr = ncu_traffic(KERNEL_OF.get(stage, stage))
    out = {"bound": "hbm", "kernel": KERNEL_OF.get(stage, stage), "stage": stage,
           "achieved": round(achieved, 1), "peak": peak, "peak_source": src, "unit": "GB/s",
           "frac": round(achieved / peak, 4),
           "traffic": tr["dram_bytes_per_launch"] if tr else None,
           "traffic_source": tr["source"] if tr else None,
           "algorithmic_bytes_per_step": int(b), "ms_per_step": round(ms, 3),
           "launches_per_step": launches}
    if stage == "composite" and evals_per_frame:
        # the compositor is issue-bound, not HBM-bound: every pixel evaluation
        # needs one ex2 on the SFU, the scarcest pipe it uses
        ev = evals_per_frame * a.frames / (ms / 1e3)
        pk = MUFU_EX2_PER_CLK_SM * SMS * SM_MHZ_MAX * 1e6
        out["compute"] = {"unit": "pixel-evals/s", "achieved": round(ev, 1),
                          "peak": pk, "peak_basis": "SFU ex2: 16/clk/SM x 148 SMs x 1965 MHz",
                          "frac": round(ev / pk, 4),
                          "evals_per_frame": int(evals_per_frame),
                          "evals_source": "CPU oracle composite of frame 0 (same splats, same order)"}
    return out


# ---------------------------------------------------------------------------
def cpu_reference(a, threads, samples, rank_seed=1002):
    """Oracle (CPU restatement) on a bounded sample: decode group 0 (all its
    frames, layers <= k) + render `samples` frames, `threads` host threads."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O
    blobs, _ = make_inputs(a, rank_seed)
    data = blobs[a.codec]
    cam = camera(a)
    info = O.read_structure(data)
    t0 = time.perf_counter()
    vals = O.decode_group_codes(data, info, 0, a.k)
    frames = O.assemble(info, info.groups[0], vals, a.k)
    t_dec = time.perf_counter() - t0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(lambda g: O.render_set(g, cam), frames[:samples]))
    t_ren = time.perf_counter() - t0
    gframes = info.groups[0].frame_count
    per_frame = t_dec / gframes + t_ren / samples
    return 1.0 / per_frame, {"decode_group_s": t_dec, "render_s": t_ren,
                             "sample": f"group 0 range/raw decode of {gframes} frames at k={a.k} "
                                       f"(amortised) + render of {samples} frames at "
                                       f"{a.width}x{a.height}, {threads} threads"}


def oracle_evals(a, rank_seed=1002):
    """Pixel evaluations (in-rect, T >= 1e-4) of frame 0 by the CPU oracle:
    the useful work of the compositor, for its compute roofline."""
    from oracle import oracle as O
    blobs, _ = make_inputs(a, rank_seed)
    data = blobs[a.codec]
    info = O.read_structure(data)
    vals = O.decode_group_codes(data, info, 0, a.k)
    f0 = O.assemble(info, info.groups[0], vals, a.k)[0]
    means, covs, depth, colors, opac, rects, _ = O.project_set(f0, camera(a))
    _, ev = O.composite(means, covs, depth, colors, opac, rects, camera(a), want_evals=True)
    return ev


def main():
    a = parse()
    a.evals_per_frame = None
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as td
        backend = "nccl" if a.impl == "b200" and torch.cuda.is_available() else "gloo"
        # GSV_BENCH_BACKEND=gloo: dev check of the multi-rank path with ranks
        # sharing one GPU (NCCL needs one GPU per rank)
        backend = os.environ.get("GSV_BENCH_BACKEND", backend)
        if a.impl == "b200" and torch.cuda.is_available():
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
        td.init_process_group(backend=backend)
        dist = td
    if a.impl == "reference":
        if rank == 0:
            threads = len(os.sched_getaffinity(0))
            samples = max(a.cpu_sample_frames, min(threads, 8))
            fps, det = cpu_reference(a, threads, samples)
            line = {"metric": METRIC, "value": round(fps, 4), "unit": "frames/s",
                    "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
                    "ms_per_step": round(1e3 / fps, 2), "higher_is_better": True,
                    "scaling": "weak", "vs_baseline": None, "dtype": "fp64",
                    "data": "synthetic (same recipe as the b200 arm)", "impl": "reference",
                    "config": {"workload": "config2: 300k Gaussians, 6 layers, 300 frames, 1080p",
                               "k": a.k, "codec": a.codec},
                    "cpu_baseline": {"value": round(fps, 4), "unit": "frames/s", "cores": threads,
                                     "kind": "port", "sample": det["sample"]},
                    "e2e": {"value": round(fps, 4), "unit": "frames/s", "h2d_bytes_per_step": 0,
                            "d2h_bytes_per_step": 0}}
            print(json.dumps(line), flush=True)
        if dist:
            dist.destroy_process_group()
        return
    if rank == 0 and not a.no_cpu:
        try:
            a.evals_per_frame = oracle_evals(a)
        except Exception as e:  # noqa: BLE001
            print(f"[bench] oracle eval count unavailable: {e}", file=sys.stderr)
    res = run_b200(a, rank, world, dist)
    if rank == 0:
        if not a.no_cpu:
            fps, det = cpu_reference(a, 1, a.cpu_sample_frames)
            res["cpu_baseline"] = {"value": round(fps, 4), "unit": "frames/s", "cores": 1,
                                   "kind": "port", "sample": det["sample"]}
        print(json.dumps(res), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
