"""Summarise an ncu --metrics gpu__time_duration.sum launch list (dev tool)."""
import collections
import csv
import sys


def summary(path, frames=4):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        k = d['Kernel Name'].split('(')[0][:44]
        agg[k][0] += 1
        agg[k][1] += float(d['Metric Value'])
    tot = sum(v[1] for k, v in agg.items() if 'crc' not in k and 'rc_decode' not in k)
    print(f"{path}: render kernels per frame {tot / 1e3 / frames:.1f} us")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"   {k:44s} n={n:4d} total={v / 1e3:9.1f}us avg={v / n / 1e3:8.2f}us "
              f"per-frame={v / 1e3 / frames:7.1f}us")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summary(p)
