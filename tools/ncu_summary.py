"""Key metrics of an ncu report (first profiled kernel of each name) as a table / JSON."""
import csv
import json
import subprocess
import sys

WANT = ["Duration", "Elapsed Cycles", "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Avg. Active Threads Per Warp",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "DRAM Throughput", "Memory Throughput",
        "Compute (SM) Throughput", "Waves Per SM", "No Eligible", "Branch Efficiency", "Grid Size", "Block Size"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mi, ui, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    res = {}
    for r in rows[1:]:
        if r[ii] != rows[1][ii]:
            continue
        if r[mi] in WANT:
            res[f"{r[mi]} [{r[ui]}]"] = r[vi]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hh = rr[0]
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
                 "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
                 "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "lts__t_sectors.sum",
                 "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"):
        if name in hh:
            j = hh.index(name)
            res[f"{name} [{rr[1][j]}]"] = rr[2][j]
    return res


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        s = summary(rep)
        print(rep)
        for k, v in s.items():
            print(f"  {k:60s} {v}")
