#!/usr/bin/env python3
"""One-screen summary of an ncu report: time, DRAM, pipes, smem wavefronts and
bank conflicts, occupancy, stall reasons."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    for row in r[2:]:
        d = dict(zip(r[0], row))
        print("==", d.get("Kernel Name", "")[:80])
        for k in KEYS:
            if k in d:
                print(f"  {k:80s} {d[k]}")
        st = {h[len('smsp__pcsamp_warps_issue_stalled_'):]: float(v or 0) for h, v in d.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
        tot = sum(st.values()) or 1.0
        print("  stalls:", ", ".join(f"{k} {v / tot:.2f}" for k, v in
                                     sorted(st.items(), key=lambda t: -t[1])[:8]))


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)
