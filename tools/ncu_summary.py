"""Key metrics per kernel from an ncu --set full report (read here, no GPU).

    python tools/ncu_summary.py gpurun_out/frame.ncu-rep
Prints a markdown table; the stall columns are the top warp-state samples."""
import csv
import subprocess
import sys

METRICS = [
    ("duration us", "gpu__time_duration.sum", 1.0),
    ("DRAM read MB", "dram__bytes_read.sum", 1.0),
    ("DRAM write MB", "dram__bytes_write.sum", 1.0),
    ("regs", "launch__registers_per_thread", 1.0),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    ("tensor pipe %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("fp64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("L1TEX %", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1.0),
    ("L2 %", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("L1 hit %", "l1tex__t_sector_hit_rate.pct", 1.0),
    ("L2 hit %", "lts__t_sector_hit_rate.pct", 1.0),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2:]


def stalls(hdr, row, top=4):
    pre = "smsp__average_warp_latency_issue_stalled_"
    pairs = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                pairs.append((float(row[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    pairs.sort(reverse=True)
    return ", ".join(f"{n} {v:.2f}" for v, n in pairs[:top])


def main():
    hdr, units, data = rows(sys.argv[1])
    cols = ["kernel"] + [m[0] for m in METRICS] + ["top stalls (warps per issue)"]
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for row in data:
        name = row[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        vals = []
        for _, key, _s in METRICS:
            if key in hdr:
                v = row[hdr.index(key)]
                u = units[hdr.index(key)]
                try:
                    f = float(v.replace(",", ""))
                    f *= {"byte": 1e-6, "Kbyte": 1e-3, "Gbyte": 1e3, "ms": 1e3,
                          "msecond": 1e3, "ns": 1e-3, "nsecond": 1e-3}.get(u, 1.0)
                    vals.append(f"{f:.1f}")
                except ValueError:
                    vals.append(v)
            else:
                vals.append("-")
        print("| " + " | ".join([name] + vals + [stalls(hdr, row)]) + " |")


if __name__ == "__main__":
    main()
