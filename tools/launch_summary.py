"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel name.

usage: python tools/launch_summary.py launches.csv [header comment ...] > profiles/rNN/launches_x.txt
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    rows = [r for r in csv.reader(open(path)) if r]
    head = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[head]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    idi = h.index("ID")
    per = collections.OrderedDict()
    for r in rows[head + 1:]:
        if len(r) < len(h):
            continue
        name = r[ki].split("(")[0][:50]
        d = per.setdefault(name, {}).setdefault(r[idi], {})
        d[r[mi]] = float(r[vi].replace(",", ""))
    for c in sys.argv[2:]:
        print("# " + c)
    print(f"{'kernel':50s} {'launches':>8s} {'avg_us':>10s} {'share':>7s}")
    tot = sum(sum(m.get("gpu__time_duration.sum", 0) for m in ls.values()) for ls in per.values())
    for name, ls in per.items():
        t = [m.get("gpu__time_duration.sum", 0) for m in ls.values()]
        # ncu reports gpu__time_duration in ns (usecond when the unit column says so)
        print(f"{name:50s} {len(t):8d} {sum(t) / len(t) / 1e3:10.1f} {sum(t) / tot * 100:6.1f}%")


if __name__ == "__main__":
    main()
