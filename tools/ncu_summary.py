#!/usr/bin/env python
"""Summarize an ncu report (--set full) or a launch-list CSV into a short text table.

    python tools/ncu_summary.py report.ncu-rep          # per-kernel key counters + top stall reasons
    python tools/ncu_summary.py --launches launches.csv # per-kernel device time share of a launch list
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_inst_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_registers", "blk_lim_regs"),
    ("launch__occupancy_limit_shared_mem", "blk_lim_smem"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "ffma_thread_inst"),
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarize(report):
    hdr, units, rows = raw(report)
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
             and h.endswith("_per_issue_active.ratio")]
    for r in rows:
        print("=" * 100)
        print(r[hdr.index("Kernel Name")][:120])
        for key, name in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"  {name:16s} {r[i]:>16s} {units[i]}")
        # tensor-pipe utilisation (tcgen05 kernels): every sm__pipe_tensor* / *tmem* percentage the report has
        for i, h in enumerate(hdr):
            if ("pipe_tensor" in h or "tmem" in h.lower() or "pipe_uniform" in h) and "pct" in h and r[i]:
                print(f"  {h[:70]:70s} {r[i]:>10s}")
        vals = sorted(((float(r[i] or 0), hdr[i]) for i in stall), reverse=True)[:6]
        tot = sum(float(r[i] or 0) for i in stall)
        print("  stalls (warps per issue):", ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
            for v, h in vals), f"(total {tot:.2f})")


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
              "second": 1e3, "s": 1e3}[r[ui]]
        name = r[ki].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'avg ms':>10s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:10.3f} {tot[k] / cnt[k]:10.3f} {tot[k] / s:7.1%}")
    print(f"{'total':60s} {sum(cnt.values()):8d} {s:10.3f}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        summarize(sys.argv[1])
