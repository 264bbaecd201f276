#!/usr/bin/env python
"""Add a kernel's measured DRAM bytes per element to profiles/quant_traffic.json
from an ncu CSV launch list (dram__bytes_read.sum / dram__bytes_write.sum per
launch), summed over every listed quant_kernel launch.

    python tools/traffic_entry.py KEY launches.csv ELEMENTS "kernel" "source"
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    key, path, elements, kernel, source = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4], sys.argv[5]
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = wr = 0.0
    n = 0
    for r in rows[1:]:
        if "quant_kernel" not in r[ki]:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        if r[mi] == "dram__bytes_read.sum":
            rd += v
            n += 1
        elif r[mi] == "dram__bytes_write.sum":
            wr += v
    f = os.path.join(ROOT, "profiles", "quant_traffic.json")
    d = json.load(open(f))
    d[key] = {"kernel": kernel, "source": source, "launches": n, "elements": elements,
              "dram_bytes_read": rd, "dram_bytes_write": wr,
              "dram_bytes_per_elem": (rd + wr) / elements, "algorithmic_bytes_per_elem": 5.0625}
    json.dump(d, open(f, "w"), indent=1)
    print(json.dumps(d[key]))


if __name__ == "__main__":
    main()
