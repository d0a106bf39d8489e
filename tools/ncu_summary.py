"""Summarise one kernel of an ncu --set full report into metric,unit,value
CSV rows (the metrics DESIGN.md and bench.py cite).

    python tools/ncu_summary.py gpurun_out/k1.ncu-rep [updates_per_launch] > profiles/X.csv
"""
import csv
import io
import subprocess
import sys

METRICS = [
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "launch__block_size",
    "launch__grid_size", "launch__occupancy_limit_registers", "launch__registers_per_thread",
    "sm__cycles_elapsed.avg.per_second", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
]


def main(rep, upl=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, vals = rows[0], rows[1], rows[2]
    w = csv.writer(sys.stdout)
    w.writerow(["metric", "unit", "value"])
    w.writerow(["kernel", "", vals[head.index("Kernel Name")] if "Kernel Name" in head else ""])
    for m in METRICS:
        if m in head:
            i = head.index(m)
            w.writerow([m, units[i], vals[i].replace(",", "")])
    if upl:
        w.writerow(["updates_per_launch", "", upl])


if __name__ == "__main__":
    main(*sys.argv[1:])
