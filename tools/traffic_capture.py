"""DRAM traffic per launch of every kernel in an ncu launch list, as the `traffic` of the bench
roofline objects (profiles/ncu_traffic.json, read by bench.py).

usage: python tools/traffic_capture.py launches.csv [out.json]
launches.csv: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
              --clock-control none --csv --log-file launches.csv python bench.py ...
Kernel names are normalised as bench.py names them: no `void `, no anonymous namespace, no
parameter list (template arguments kept).  Per kernel: mean dram read + write bytes per launch.
"""
import collections
import csv
import json
import re
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def norm(name):
    name = name.replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    depth, out = 0, []
    for ch in name:  # cut at the parameter list: the first '(' outside template brackets
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0:
            break
        out.append(ch)
    return re.sub(r"\s+", " ", "".join(out)).strip()


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if r]
    head = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[head]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    per = collections.defaultdict(lambda: collections.defaultdict(dict))
    for r in rows[head + 1:]:
        if len(r) < len(h):
            continue
        v = float(r[vi].replace(",", ""))
        if ui is not None and r[mi].startswith("dram__bytes"):
            v *= UNITS.get(r[ui], 1)
        per[norm(r[ki])][r[idi]][r[mi]] = v
    out = {"_source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                      "--clock-control none (%s): mean dram read + write bytes per launch" % sys.argv[1]}
    for name, launches in per.items():
        t = [m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in launches.values()]
        if t:
            out[name] = int(sum(t) / len(t))
    js = json.dumps(out, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(js + "\n")
    print(js)


if __name__ == "__main__":
    main()
