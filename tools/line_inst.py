"""Per-source-line executed warp instructions from
`ncu --page source --csv --print-source=cuda,sass` output (SASS rows)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur = None
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name":
        continue
    if cur and hdr and r[0].isdigit() and len(r) > 8 and r[2] == "-":
        try:
            inst = int(r[7] or 0)
        except ValueError:
            continue
        key = (cur, int(r[0]))
        a = agg.setdefault(key, [0, r[1].strip()[:90]])
        a[0] += inst
tot = sum(v[0] for v in agg.values()) or 1
print("warp instructions", tot)
for (f, ln), (i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100 * i / tot:5.1f}% {i:>12d} {f}:{ln:<5d} {src}")
