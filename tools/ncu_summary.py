"""Condense an .ncu-rep into the handful of numbers DESIGN.md / profiles/ cite.
    python tools/ncu_summary.py gpurun_out/k1.ncu-rep [--out profiles/r01_k1.txt]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
    "sass__inst_executed_shared_loads", "sass__inst_executed_shared_stores", "sass__inst_executed_global_loads",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
]
STALL = "smsp__average_warps_issue_stalled_"


def main():
    rep = sys.argv[1]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    hdr, units = rows[0], rows[1]
    lines = []
    for data in rows[2:]:
        rec = dict(zip(hdr, zip(units, data)))
        lines.append(f"== kernel {rec.get('Kernel Name', ('', '?'))[1]}  (id {rec.get('ID', ('', '?'))[1]})")
        for k in KEYS:
            if k in rec:
                lines.append(f"{k} = {rec[k][1]} {rec[k][0]}")
        stalls = [(float(v[1] or 0), k[len(STALL):].replace('_per_issue_active.ratio', '')) for k, v in rec.items()
                  if k.startswith(STALL) and k.endswith("per_issue_active.ratio")]
        lines.append("stall reasons (warps per issue-active cycle): " +
                     ", ".join(f"{n}={x:.2f}" for x, n in sorted(stalls, reverse=True)[:8]))
    body = "\n".join(lines)
    print(body)
    if out:
        with open(out, "w") as f:
            f.write(f"# condensed from {rep} by tools/ncu_summary.py (ncu --set full --clock-control none)\n" + body + "\n")


if __name__ == "__main__":
    main()
