"""Aggregate an ncu launch list (csv: gpu__time_duration[, dram bytes]) into per-kernel shares.

Usage: launch_share.py launches.csv [steps]  -> prints a table and writes a json next to it."""
import csv
import io
import json
import re
import sys
from collections import OrderedDict


def main(path, steps=1):
    txt = open(path).read()
    lines = [l for l in txt.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    data = rows[1:]
    ki = hdr.index("Kernel Name")
    mi = hdr.index("Metric Name")
    vi = hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    ii = hdr.index("ID")
    per = OrderedDict()
    launches = {}
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "byte": 1.0, "B": 1.0,
             "KB": 1e3, "MB": 1e6, "GB": 1e9, "Kbyte": 1e3, "Mbyte": 1e6,
             "Gbyte": 1e9}
    for r in data:
        name = re.sub(r"\(pcb::PassArgs\)|void |pcb::|\(anonymous namespace\)::|<unnamed>::", "", r[ki]).strip()
        key = (r[ii], name)
        launches.setdefault(key, {})[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    for (lid, name), m in launches.items():
        base = name.split("<")[0]
        d = per.setdefault(name, {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
        d["launches"] += 1
        d["ms"] += m.get("gpu__time_duration.sum", 0.0)
        d["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(d["ms"] for d in per.values()) or 1.0
    print(f"{'kernel':44s} {'launches':>8s} {'ms/step':>9s} {'share':>6s} {'dram GB/step':>12s}")
    for name, d in sorted(per.items(), key=lambda kv: -kv[1]["ms"]):
        print(f"{name[:44]:44s} {d['launches'] / steps:8.1f} {d['ms'] / steps:9.3f} {d['ms'] / tot:6.1%} "
              f"{d['dram_bytes'] / steps / 1e9:12.3f}")
    out = {name: {"launches_per_step": d["launches"] / steps, "ms_per_step": d["ms"] / steps,
                  "share": d["ms"] / tot, "dram_bytes_per_step": d["dram_bytes"] / steps}
           for name, d in per.items()}
    with open(path.rsplit(".", 1)[0] + "_share.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
