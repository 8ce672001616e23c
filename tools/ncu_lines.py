"""Executed warp instructions and stall samples per source line, with the
opcode mix of each line, from an ncu report (read here, no GPU):

    [NCU_KERNEL=regex:name] python tools/ncu_lines.py report.ncu-rep [top]
Joins `--page source --print-source=sass` (per-instruction counts) with the
`cuda,sass` view (address -> source line)."""
import collections
import csv
import os
import subprocess
import sys


def export(rep, view):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=" + view]
    if os.environ.get("NCU_KERNEL"):  # e.g. NCU_KERNEL=regex:k_trace for multi-kernel reports
        cmd += ["-k", os.environ["NCU_KERNEL"]]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    addr2line = {}
    cur = None
    line = None
    for r in export(rep, "cuda,sass"):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0].isdigit() and len(r) > 2 and r[2] == "-":
            line = (cur, int(r[0]), r[1].strip()[:60])
        elif len(r) > 2 and r[0] == "" and r[2].startswith("0x") and line:
            addr2line[r[2]] = line
    per = collections.defaultdict(lambda: [0, 0, collections.Counter()])
    tot = 0
    for r in export(rep, "sass")[2:]:
        if len(r) < 6 or not r[0].startswith("0x"):
            continue
        try:
            ie, st = int(r[5]), int(r[2])
        except ValueError:
            continue
        toks = r[1].strip().split()
        op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?"))
        key = addr2line.get(r[0], ("?", 0, ""))
        a = per[key]
        a[0] += ie
        a[1] += st
        a[2][op.split(".")[0]] += ie
        tot += ie
    print("executed warp instructions", tot)
    for (f, ln, src), (n, s, ops) in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
        mix = " ".join(f"{o}:{c * 100 // max(n, 1)}" for o, c in ops.most_common(4))
        print(f"{100 * n / tot:5.1f}% st{s:6d} {f}:{ln:<5d} {src:60s} [{mix}]")


if __name__ == "__main__":
    main()
