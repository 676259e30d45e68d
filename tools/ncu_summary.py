"""Summarise an .ncu-rep: key SOL/occupancy/scheduler metrics + SASS opcode mix and hottest stalls."""
import collections, csv, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
keep = ("Duration", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Issued Instructions", "Avg. Active Threads Per Warp", "Block Limit Shared Mem", "Block Limit Registers",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "Waves Per SM")
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in keep:
        print(f"{d['Kernel Name'][:30]:30s} {d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
if len(rr) > 2:
    h = rr[0]
    for r in rr[2:]:
        d = dict(zip(h, r))
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed_pipe_fp64.sum",
                  "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
                  "sm__sass_thread_inst_executed_op_dmul_pred_on.sum"):
            if k in d:
                print(f"raw {k:60s} {d[k]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
if len(rows) > 2:
    hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
    tot = 0; byop = collections.Counter(); stall = collections.Counter(); hot = []
    for r in rows[2:]:
        if len(r) < len(hdr): continue
        try: ie = int(r[idx["Instructions Executed"]] or 0)
        except ValueError: continue
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        srcl = r[idx["Source"]].strip()
        toks = srcl.split()
        op = (toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")).split(".")[0]
        byop[op] += ie; stall[op] += s; tot += ie
        hot.append((s, ie, srcl))
    print("instructions executed", tot)
    for op, n in byop.most_common(18):
        print(f"  {op:8s} {n:11d} {100*n/tot:5.1f}%  stall-samples {stall[op]}")
    print("hottest (stall samples, exec count, sass):")
    for s, ie, t in sorted(hot, reverse=True)[:25]:
        print(f"  {s:6d} {ie:9d}  {t[:90]}")
