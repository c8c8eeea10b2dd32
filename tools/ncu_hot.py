"""Top SASS lines by warp-stall samples and stall-reason totals of one ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, v = r[0], r[2]
want = ["gpu__time_duration.sum", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]
for w in want:
    if w in h:
        print(f"{w:80s} {v[h.index(w)]}")
st = []
for i, x in enumerate(h):
    if x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued"):
        try:
            st.append((float(v[i].replace(",", "")), x.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(a for a, _ in st) or 1
print("stalls:", ", ".join(f"{x} {100*a/tot:.1f}%" for a, x in sorted(st, reverse=True)[:9]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hh = rows[1]
ia, isrc, isamp = hh.index("Address"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
data = []
for rr in rows[2:]:
    try:
        data.append((int(rr[isamp] or 0), rr[ia][-5:], rr[isrc][:90]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for d in sorted(data, reverse=True)[:top]:
    print(f"{100*d[0]/tot:5.1f}% {d[1]} {d[2]}")
