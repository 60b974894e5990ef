"""Print selected metrics of one or more `ncu --page raw --csv` dumps side by side.
usage: python tools/ncu_raw.py a.csv [b.csv ...]"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]


def load(f):
    rows = list(csv.reader(open(f)))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


ds = [load(f) for f in sys.argv[1:]]
for k in KEYS:
    print("%-78s %s" % (k, "  ".join("%s %s" % d.get(k, ("-", "")) for d in ds)))
