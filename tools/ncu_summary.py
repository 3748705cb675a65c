#!/usr/bin/env python
"""Summarise an ncu --set full report and an ncu launch list (CSV) into markdown.

    python tools/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv ALG_BYTES_PER_LAUNCH > summary.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def to_bytes(val, unit):
    f = float(val)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    report, launches, alg = sys.argv[1], sys.argv[2], float(sys.argv[3])
    d = raw(report)
    print(f"# ncu summary: `{d.get('Kernel Name', ('ar_exec_kernel', ''))[0]}`\n")
    print("| metric | value |\n|---|---|")
    for k, name in KEYS:
        if k in d:
            print(f"| {name} (`{k}`) | {d[k][0]} {d[k][1]} |")
    rd = to_bytes(*d["dram__bytes_read.sum"])
    wr = to_bytes(*d["dram__bytes_write.sum"])
    print(f"| traffic = read + write | {(rd + wr) / 1e9:.4f} GB |")
    print(f"| algorithmic bytes per launch | {alg / 1e9:.4f} GB |")
    print(f"| traffic / algorithmic | {(rd + wr) / alg:.4f} |")
    stalls = [(k, float(v[0])) for k, v in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    stalls.sort(key=lambda x: -x[1])
    print("\nTop warp stall reasons (warps per issue-active cycle):\n")
    for k, v in stalls[:6]:
        print(f"* `{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}`: {v:.3f}")
    # launch list shares
    rows = [r for r in csv.reader(open(launches)) if r and not r[0].startswith("==")]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot = {}
    for r in rows[1:]:
        tot.setdefault(r[ki].split("(")[0], []).append(float(r[vi]))
    allns = sum(sum(v) for v in tot.values())
    print("\nLaunch list (`--metrics gpu__time_duration.sum --clock-control none`, cold, serialised):\n")
    print("| kernel | launches | mean duration | share of listed time |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} us | {sum(v) / allns * 100:.1f} % |")


if __name__ == "__main__":
    main()
