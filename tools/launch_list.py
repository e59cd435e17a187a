"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list.
Usage: python tools/launch_list.py launches.csv [--order]"""
import csv
import re
import sys
from collections import OrderedDict


def short(name: str) -> str:
    name = re.sub(r"\(anonymous namespace\)::", "", name)
    name = re.sub(r"\(.*\)$", "", name)  # drop the argument list
    return name.replace("void ", "")


def load(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for rec in csv.DictReader(lines):
        if rec.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(rec["Metric Value"].replace(",", ""))
        unit = rec["Metric Unit"]
        us = v / 1e3 if unit == "ns" else v if unit == "us" else v * 1e3 if unit == "ms" else v
        rows.append((short(rec["Kernel Name"]), rec["Grid Size"], rec["Block Size"], us))
    return rows


def main():
    rows = load(sys.argv[1])
    total = sum(r[3] for r in rows)
    print(f"launches {len(rows)}, total {total:.1f} us")
    agg = OrderedDict()
    for name, _, _, us in rows:
        a = agg.setdefault(name, [0.0, 0])
        a[0] += us
        a[1] += 1
    for name, (us, cnt) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{us:9.1f} us {100 * us / total:5.1f}%  x{cnt:<3d} {name}")
    if "--order" in sys.argv:
        print("\nin launch order:")
        for i, (name, grid, block, us) in enumerate(rows):
            print(f"{i:4d} {us:9.1f} us  grid {grid:>14s} block {block:>12s}  {name}")


if __name__ == "__main__":
    main()
