"""Markdown summary of ncu --page raw --csv exports (tools only).

    python tools/ncu_summary.py title out.md name=path.raw.csv [name=path.raw.csv ...]

One column per capture; the metrics below, and for kernels with the executed
FP32 counters the executed flops (2 FFMA + FADD + FMUL + 4 FFMA2 + 2 FMUL2 +
2 FADD2) per launch.
"""
import csv
import sys

METRICS = [
    "Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_static", "dram__bytes_read.sum", "dram__bytes_write.sum",
]
FP = {"smsp__sass_thread_inst_executed_op_ffma_pred_on.sum": 2, "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum": 1,
      "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum": 1, "smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum": 4,
      "smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum": 2, "smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum": 2}


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def main():
    title, out = sys.argv[1], sys.argv[2]
    cols = []
    for arg in sys.argv[3:]:
        name, path = arg.split("=", 1)
        for d, u in load(path):
            cols.append((name, d, u))
    lines = [f"# {title}", "", "| metric | unit | " + " | ".join(c[0] for c in cols) + " |",
             "|---|---|" + "---|" * len(cols)]
    for m in METRICS + list(FP):
        unit = next((c[2].get(m, "") for c in cols if m in c[2]), "")
        lines.append(f"| `{m}` | {unit} | " + " | ".join(c[1].get(m, "—") for c in cols) + " |")
    lines.append("")
    for name, d, _ in cols:
        if all(k in d for k in FP):
            ex = sum(float(d[k].replace(",", "")) * w for k, w in FP.items())
            lines.append(f"- {name}: executed FP32 flops per launch {ex:.4e}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
