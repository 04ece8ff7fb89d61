"""Dev analysis: how many (splat, tile) pairs of a config-2 frame can hold a
pixel whose alpha reaches eps (the rest contribute below eps to every pixel
of the tile), and how many rect pixels do.  Oracle projection of frame 0.

usage: cull_stats.py [container.gsv]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from oracle import oracle as O
from paper_2509_17513_b200.configs import axis_camera

path = sys.argv[1] if len(sys.argv) > 1 else "/tmp/gsv_bench_cache/85ece8f9d20f426a_c0.gsv"
data = open(path, "rb").read()
info = O.read_structure(data)
vals = O.decode_group_codes(data, info, 0, info.layer_count)
gset = O.assemble(info, info.groups[0], vals, info.layer_count, only=[0])[0]
cam = axis_camera(1920, 1080)
means, cov, depth, colors, opac, rects, idx = O.project_set(gset, cam)
n = len(means)
det = cov[:, 0, 0] * cov[:, 1, 1] - cov[:, 0, 1] * cov[:, 1, 0]
ia, ib, ic = cov[:, 1, 1] / det, -cov[:, 0, 1] / det, cov[:, 0, 0] / det
print(f"{n} splats, rect pixels {int(((rects[:, 1] - rects[:, 0]) * (rects[:, 3] - rects[:, 2])).sum()):,}")


def min_q(ia, ib, ic, x0, x1, y0, y1):
    """min over integer-box corners/edges (continuous relaxation) of
    q = ia dx^2 + 2 ib dx dy + ic dy^2 with dx in [x0, x1], dy in [y0, y1]."""
    inside = (x0 <= 0) & (x1 >= 0) & (y0 <= 0) & (y1 >= 0)
    best = np.full(ia.shape, np.inf)
    for fixed_x in (x0, x1):  # dx fixed, dy free in [y0, y1]: dy* = -ib dx / ic
        dy = np.clip(-ib * fixed_x / ic, y0, y1)
        best = np.minimum(best, ia * fixed_x ** 2 + 2 * ib * fixed_x * dy + ic * dy ** 2)
    for fixed_y in (y0, y1):
        dx = np.clip(-ib * fixed_y / ia, x0, x1)
        best = np.minimum(best, ia * dx ** 2 + 2 * ib * dx * fixed_y + ic * fixed_y ** 2)
    return np.where(inside, 0.0, best)


pairs, keep = 0, {e: 0 for e in (1e-4, 1e-6, 1e-7, 1e-8)}
pix_keep = {e: 0 for e in keep}
T = 16
for s in range(0, n, 20000):
    sl = slice(s, min(n, s + 20000))
    r = rects[sl]
    tx0, tx1 = r[:, 0] // T, (r[:, 1] - 1) // T
    ty0, ty1 = r[:, 2] // T, (r[:, 3] - 1) // T
    for i in range(r.shape[0]):
        j = s + i
        txs = np.arange(tx0[i], tx1[i] + 1)
        tys = np.arange(ty0[i], ty1[i] + 1)
        gx, gy = np.meshgrid(txs, tys)
        gx, gy = gx.ravel(), gy.ravel()
        bx0 = np.maximum(gx * T, r[i, 0]) - means[j, 0]
        bx1 = np.minimum(gx * T + T, r[i, 1]) - 1 - means[j, 0]
        by0 = np.maximum(gy * T, r[i, 2]) - means[j, 1]
        by1 = np.minimum(gy * T + T, r[i, 3]) - 1 - means[j, 1]
        q = min_q(ia[j], ib[j], ic[j], bx0, bx1, by0, by1)
        amax = opac[j] * np.exp(-0.5 * q)
        pairs += q.size
        for e in keep:
            keep[e] += int((amax >= e).sum())
    if s % 100000 == 0:
        print(f"  {s}/{n}", flush=True)
print(f"(splat, tile) pairs {pairs:,}")
for e, k in keep.items():
    print(f"  eps {e:g}: pairs holding alpha >= eps {k:,} ({k / pairs:.3f})")
