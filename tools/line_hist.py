"""Per-source-line stall histogram from
`ncu --page source --csv --print-source=cuda,sass` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur = None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if cur and r[0].isdigit() and len(r) > 6 and r[2] == "-":
        try:
            s = int(r[4] or 0)
            e = int(r[7] or 0)
        except ValueError:
            continue
        key = (cur, int(r[0]))
        a = agg.setdefault(key, [0, 0, r[1].strip()[:80]])
        a[0] += s
        a[1] += e
tot = sum(v[0] for v in agg.values()) or 1
print("stall samples", tot)
for (f, ln), (s, e, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5d} {src}")
