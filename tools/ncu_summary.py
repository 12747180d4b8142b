"""Summarize an ncu report: per kernel duration, DRAM bytes/throughput,
occupancy, registers, bank conflicts, FP64 pipe and the top warp stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_") and
              h.endswith("_per_issue_active.ratio")]
name_i = hdr.index("Kernel Name")
for r in rows[2:]:
    print("----", r[name_i][:90])
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:65s} {r[i]} {units[i]}")
    st = []
    for i in stall_cols:
        try:
            st.append((float(r[i]), hdr[i]))
        except ValueError:
            pass
    st.sort(reverse=True)
    for v, h in st[:6]:
        print(f"  stall {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):40s} {v:.1f}")
