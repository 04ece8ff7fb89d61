"""Summarise ncu --set full reports: time, DRAM bytes, occupancy, top stall reasons (dev tool)."""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"),
        ("dram__bytes_write.sum", "dram_wr"), ("launch__registers_per_thread", "regs"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
        ("smsp__inst_executed.sum", "inst"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("l1tex__t_bytes.sum", "l1_bytes"), ("lts__t_bytes.sum", "l2_bytes")]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def summary(path):
    hdr, units, rows = raw(path)
    for r in rows:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"== {d['Kernel Name'][:70]}")
        print("   " + "  ".join(f"{n}={d.get(k, '?')}{u.get(k, '')}" for k, n in KEYS if k in d))
        stalls = [(k, float(d[k])) for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled_")
                  and k.endswith(".ratio") and d.get(k, "").replace(".", "").isdigit()]
        if not stalls:
            stalls = [(k, float(d[k].replace(',', ''))) for k in hdr
                      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")
                      and d.get(k, "").replace(",", "").replace(".", "").isdigit()]
        stalls.sort(key=lambda x: -x[1])
        print("   stalls: " + ", ".join(f"{k.split('stalled_')[1].replace('.ratio', '')}={v:.2f}"
                                       for k, v in stalls[:7]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summary(p)
