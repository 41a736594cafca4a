#!/usr/bin/env python3
"""Summarise an ncu report: key throughput metrics, stall reasons, hot SASS."""
import csv, subprocess, sys, io

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2] if len(r) > 2 else r[1]))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum",
        "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum", "lts__t_bytes.sum"]

def main(rep):
    d = raw(rep)
    for k in KEYS:
        for h, v in d.items():
            if h == k:
                print(f"{k:70s} {v}")
    st = {h: v for h, v in d.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
    tot = sum(float(v or 0) for v in st.values())
    print("stall samples (share):")
    for h, v in sorted(st.items(), key=lambda x: -float(x[1] or 0))[:8]:
        print(f"   {h.replace('smsp__pcsamp_warps_issue_stalled_',''):30s} {float(v)/tot:.3f}")

if __name__ == "__main__":
    main(sys.argv[1])
