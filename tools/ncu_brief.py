"""Key metrics + warp-stall breakdown of one kernel from an .ncu-rep (ncu --page raw --csv)."""
import csv, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]
idx = {n: i for i, n in enumerate(h)}
for w in want:
    if w in idx: print(f"{w:70s} {v[idx[w]]} {u[idx[w]]}")
st = []
for i, n in enumerate(h):
    if "pcsamp_warps_issue_stalled" in n and not n.endswith("not_issued"):
        try: st.append((float(v[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError: pass
st.sort(reverse=True)
tot = sum(x for x, _ in st) or 1
print("stalls:", ", ".join(f"{n} {100 * x / tot:.1f}%" for x, n in st[:9]))
