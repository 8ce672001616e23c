"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel.

    python tools/launch_summary.py launches.csv
Prints a markdown table: kernel, launches, total ns, mean ns, share."""
import csv
import re
import sys
from collections import OrderedDict


def summarise(path):
    rows = OrderedDict()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
        ns = float(r["Metric Value"].replace(",", ""))
        c, t = rows.get(name, (0, 0.0))
        rows[name] = (c + 1, t + ns)
    return rows


def main():
    rows = summarise(sys.argv[1])
    total = sum(t for _, t in rows.values())
    print("| kernel | launches | total ns | mean ns | share |")
    print("|---|---|---|---|---|")
    for name, (c, t) in sorted(rows.items(), key=lambda kv: -kv[1][1]):
        print(f"| {name} | {c} | {t:.0f} | {t / c:.0f} | {100 * t / total:.1f}% |")
    print(f"| **total** | {sum(c for c, _ in rows.values())} | {total:.0f} | | |")


if __name__ == "__main__":
    main()
