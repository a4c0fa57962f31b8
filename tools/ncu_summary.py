import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
r = list(csv.reader(out.splitlines()))
h, u = r[0], r[1]
keys = ["gpu__time_duration.sum","dram__bytes_read.sum","dram__bytes_write.sum","launch__registers_per_thread",
 "sm__warps_active.avg.pct_of_peak_sustained_active","sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
 "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active","smsp__inst_executed.sum","sm__throughput.avg.pct_of_peak_sustained_elapsed",
 "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed","lts__t_bytes.sum","l1tex__t_bytes.sum",
 "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum","smsp__sass_thread_inst_executed_op_dmul_pred_on.sum","smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
 "smsp__issue_active.avg.pct_of_peak_sustained_active","local_load","local_store"]
for row in r[2:]:
    d = dict(zip(h,row))
    print(d.get("Kernel Name","")[:60])
    for k in keys:
        for name in h:
            if name == k or (k in ("local_load","local_store") and k in name and name.endswith(".sum") and "l1tex__t" in name):
                print(f"   {name:75s} {d[name]} {u[h.index(name)]}")
    stalls = []
    for name in h:
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try: stalls.append((float(d[name].replace(",","")), name[33:]))
            except: pass
    tot = sum(s for s,_ in stalls)
    print("   stalls:", ", ".join(f"{n}={s/tot:.2f}" for s,n in sorted(stalls, reverse=True)[:8]))
