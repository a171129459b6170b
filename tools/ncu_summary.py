#!/usr/bin/env python
"""Summarise an ncu report: key metrics, stall reasons, SASS opcode mix.  Usage: ncu_summary.py REP"""
import collections
import csv
import io
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, top=18):
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h, v = raw[0], raw[2]
    d = dict(zip(h, v))
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed.sum.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second"]
    for k in keys:
        if k in d:
            print(f"{k:62s} {d[k]}")
    stalls = {k: float(x) for k, x in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
              and x not in ("", "n/a")}
    print("stalls (warps per issue):")
    for k, x in sorted(stalls.items(), key=lambda t: -t[1])[:8]:
        print(f"   {k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''):28s} {x:.3f}")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    hh = src[1]
    ii = hh.index("Instructions Executed"); si = hh.index("Source")
    ops = collections.Counter(); tot = 0
    for x in src[2:]:
        try:
            n = int(x[ii])
        except Exception:
            continue
        t = x[si].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[op] += n; tot += n
    print("warp instructions executed:", tot)
    print("   " + "  ".join(f"{k}:{100*v/tot:.1f}%" for k, v in ops.most_common(top)))


if __name__ == "__main__":
    main(sys.argv[1])
