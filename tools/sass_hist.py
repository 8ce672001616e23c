"""Per-opcode executed-instruction and stall-sample histogram from an
`ncu --page source --csv --print-source=sass` dump."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
i_src, i_s, i_e = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index(
    "Instructions Executed")
st, ex = defaultdict(int), defaultdict(int)
for r in rows[hi + 1:]:
    if len(r) <= i_e or not r[i_src].strip() or r[0] == "Address":
        continue
    t = r[i_src].strip().split()
    op = (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]
    try:
        st[op] += int(r[i_s] or 0)
        ex[op] += int(r[i_e] or 0)
    except ValueError:
        pass
tot, ts = sum(ex.values()) or 1, sum(st.values()) or 1
print("executed", tot, "stall samples", ts)
for op in sorted(st, key=lambda o: -st[o])[: int(sys.argv[2]) if len(sys.argv) > 2 else 16]:
    print(f"{op:12s} {100 * ex[op] / tot:5.1f}% exec {100 * st[op] / ts:5.1f}% stall")
