"""Build profiles/ncu_traffic.json (DRAM bytes per launch per kernel, max over
the captured launches) from tools/ncu_summary.py text summaries.

usage: traffic_json.py out.json summary.txt [summary.txt ...]"""
import json
import re
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def num(tok):
    m = re.match(r"([-\d.naN]+)([A-Za-z]+)", tok)
    if not m or "nan" in m.group(1).lower():
        return None
    return float(m.group(1)) * UNITS.get(m.group(2), 1)


out = {}
srcs = sys.argv[2:]
for path in srcs:
    name = None
    for line in open(path):
        if line.startswith("== "):
            name = re.sub(r"^(void )?([A-Za-z_0-9]+).*", r"\2", line[3:].strip())
        elif name and "dram_rd=" in line:
            rd = num(re.search(r"dram_rd=(\S+)", line).group(1))
            wr = num(re.search(r"dram_wr=(\S+)", line).group(1))
            if rd is None or wr is None:
                continue
            e = out.setdefault(name, {"per_launch": []})
            e["per_launch"].append(int(rd + wr))
for k, e in out.items():
    e["dram_bytes_per_launch"] = max(e["per_launch"])
    e["launches_captured"] = len(e["per_launch"])
    e["source"] = ("ncu --set full --clock-control none (" + ", ".join(srcs) + "); max over captured launches")
json.dump(dict(sorted(out.items())), open(sys.argv[1], "w"), indent=1)
print(sorted(out))
