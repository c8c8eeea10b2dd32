"""Writes profiles/ncu_summary.json from one `ncu --set full` capture of the pair kernel."""
import csv, json, subprocess, sys
rep, capture = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
m = {k: f"{v[h.index(k)]} {u[h.index(k)]}".strip() for k in keys if k in h}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
def nbytes(k):
    i = h.index(k)
    return float(v[i].replace(",", "")) * scale.get(u[i], 1)
st = []
for i, x in enumerate(h):
    if x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued"):
        try:
            st.append((float(v[i].replace(",", "")), x.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(a for a, _ in st) or 1
m["stall_sample_share"] = {x: round(a / tot, 4) for a, x in sorted(st, reverse=True)[:9]}
out = {"jacobi_sweep_kernel": {"capture": capture,
                              "dram_bytes_per_launch": nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum"),
                              "metrics": m}}
print(json.dumps(out, indent=1))
