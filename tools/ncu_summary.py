"""Summarise an .ncu-rep (raw metrics + stall reasons + top source lines)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else None
def page(p, extra=()):
    r = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))
lines = []
raw = page("raw")
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "local_load_bytes", "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "lts__t_bytes.sum",
        "launch__shared_mem_per_block_dynamic"]
for w in want:
    if w in hdr:
        i = hdr.index(w); lines.append(f"{w:60s} {vals[i]:>20s} {units[i]}")
# stall reasons
for i, h in enumerate(hdr):
    if h.startswith("smsp__average_warp_latency_issue_stalled") or h.startswith("smsp__pcsamp_warps_issue_stalled"):
        try:
            if float(vals[i].replace(",", "")) > 0: lines.append(f"{h:60s} {vals[i]:>20s} {units[i]}")
        except ValueError: pass
txt = "\n".join(lines)
print(txt)
if out: open(out, "w").write(txt + "\n")
