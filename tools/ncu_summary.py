import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr = r[0]; vals = r[2] if len(r) > 2 else r[1]
d = dict(zip(hdr, vals))
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "lts__t_bytes.sum", "launch__grid_size"]
for k in keys:
    for h in hdr:
        if h.split(" ")[0] == k:
            print(f"{k:70s} {d[h]}")
            break
st = []
for h, v in d.items():
    if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
        try: st.append((float(v), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except: pass
tot = sum(v for v, _ in st) or 1
print("stalls:", ", ".join(f"{h} {100*v/tot:.0f}%" for v, h in sorted(st, reverse=True)[:8]))
