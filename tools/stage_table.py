"""Per-stage HBM table from the round's ncu --set full captures (dev tool).

For every captured kernel: launches, average duration, DRAM bytes per launch
(dram__bytes_read.sum + dram__bytes_write.sum: the traffic ncu measured,
cold-cache and serialised), the ALGORITHMIC bytes per launch of the
config-2 workload (what the stage must move at minimum; formulas below, SURVEY
8(d) sizes), and both as GB/s against the HBM peak.

usage: stage_table.py <dir with full_*.ncu-rep>   (markdown to stdout)"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

# config 2 (300k Gaussians, 6 layers, 30-frame groups, 1080p, k = 6) --
# counts from the bench's render_stats (frame 0) and the container layout
N = 300_000                 # splats (all visible at the axis camera)
R1 = 32_768                 # ranks in the first compositing round
TILES = 8_160
PIX = 1920 * 1080
KEYS_R1 = 783_000           # (tile, splat) pairs of round 1 (ranks < R1, 23.9 tiles per splat)
KEYS_EMIT = 1_078_580       # keys of both rounds (render_stats.n_keys_emitted)
KEYS_R2 = KEYS_EMIT - KEYS_R1
RAW_C0 = 2_348_261_640      # codec-0 container bytes (payloads of all 10 groups)
CODED_C1 = 680_576_795      # codec-1 container bytes
PLANES = 1200 * 30 * 50_176 + 180 * 30 * 50_176 * 2  # decoded code planes of one open (LE bytes)

ALG = {  # kernel -> (bytes per launch, formula)
    "crc_kernel": (None, "every payload byte once (codec 0: the container; codec 1: the decoded planes)"),
    "rc_decode_kernel": (CODED_C1 + 2 * PLANES, "coded bytes + planes written + previous planes read"),
    "fold_all_kernel": (N * 184 * 31, "184 B state read + written + 29 x 184 B deltas per splat"),
    "project_kernel": (N * (26 + 64 + 12), "26 B codes in, 64 B record + 12 B depth key/index out per splat"),
    "depth_key_prep": (N * 12, "8 B depth bits in, 4 B sort key out per splat"),
    "radix_onesweep": (N * 16, "key + value read and written per element (depth passes, n = 300k)"),
    "depth_tie_fixup": (N * 8, "sorted key + index read once per splat"),
    "r1_count_kernel": (R1 * 8 + 256 * TILES * 4, "round-1 rects + the (block, tile) count matrix written"),
    "r1_scan_blocks_kernel": (2 * 256 * TILES * 4, "count matrix read + offsets written"),
    "r1_scan_tiles_kernel": (2 * TILES * 4, "tile totals read + ranges written"),
    "r1_place_kernel": (R1 * 8 + 256 * TILES * 4 + KEYS_R1 * 4, "rects + offsets read, splat index per key written"),
    "round_emit_fused": ((N - R1) * 12 + KEYS_R2 * 8, "rank->index + rect per round-2 splat, key written"),
    "keys_to_off_kernel": (KEYS_R2 * 4 + TILES * 4, "sorted tile keys read, tile offsets written"),
    "open_mask_kernel": (TILES * 8, "tile state read, mask written"),
    "composite_strip_kernel": ((KEYS_EMIT * 52 + PIX * 12) // 2,
                               "(4 B index + 48 B record) per key + 12 B per pixel, per frame / 2 launches"),
    "reset_frame_kernel": (None, "counters only"),
    "copy_planes_kernel": (None, "RAW-mode planes of range-coded runs copied"),
}


def peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        for k in ("hbm_gbs", "hbm_copy_gbs", "hbm_GBps"):
            if k in d:
                return float(d[k]), "MEASURED_PEAKS.json"
    return 6650.0, "B200_PROFILING.md fallback"


def rows(path):
    out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))

        def val(k, scale_units):
            v = float(d[k].replace(",", ""))
            return v * scale_units.get(u.get(k, ""), 1.0)
        t = val("gpu__time_duration.sum", {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3,
                                           "nsecond": 1e-9, "second": 1.0})
        bsc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
        dram = val("dram__bytes_read.sum", bsc) + val("dram__bytes_write.sum", bsc)
        name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
        res.append((name, t, dram))
    return res


def main(dirpath):
    peak, src = peak_gbs()
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    sources = defaultdict(set)
    for rep in sorted(Path(dirpath).glob("full_*.ncu-rep")):
        for name, t, dram in rows(rep):
            key = name if not (name == "crc_kernel" and "codec1" in rep.name) else "crc_kernel (codec 1 planes)"
            a = agg[key]
            a[0] += 1
            a[1] += t
            a[2] += dram
            sources[key].add(rep.name)
    print(f"# Per-stage HBM table (config 2, k = 6; peak {peak:.0f} GB/s from {src})\n")
    print("| kernel | launches | avg time | DRAM bytes/launch | DRAM GB/s | algorithmic bytes/launch | "
          "algorithmic GB/s | frac of peak | algorithmic bytes |")
    print("|---|---|---|---|---|---|---|---|---|")
    for k, (n, t, dram) in sorted(agg.items(), key=lambda kv: -kv[1][1] / kv[1][0]):
        tt, dd = t / n, dram / n
        base = k.split(" ")[0]
        alg, how = ALG.get(base, (None, ""))
        if base == "crc_kernel":
            alg = PLANES if "codec 1" in k else RAW_C0
        tstr = f"{tt * 1e3:.3f} ms" if tt >= 1e-3 else f"{tt * 1e6:.1f} us"
        ag = f"{alg / tt / 1e9:.0f}" if alg else "-"
        fr = f"{alg / tt / 1e9 / peak:.3f}" if alg else "-"
        print(f"| {k} | {n} | {tstr} | {dd / 1e6:.2f} MB | {dd / tt / 1e9:.0f} | "
              f"{(alg / 1e6) if alg else 0:.2f} MB | {ag} | {fr} | {how} |")
    print("\nDRAM bytes are ncu's measurement of one serialised, cold-cache launch; algorithmic bytes are the "
          "stage's minimum traffic.  DRAM well below algorithmic means the data was served from L2 (126 MB).")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof2")
