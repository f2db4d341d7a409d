"""Summarise an ncu report: key SOL metrics plus the top stalled SASS lines.
   python tools/ncu_summary.py gpurun_out/prof.ncu-rep [n_top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
hdr = rows[0]
want = {"Duration", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Dynamic Shared Memory Per Block", "Executed Instructions",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Avg. Active Threads Per Warp",
        "Block Limit Registers", "Block Limit Shared Mem", "Grid Size", "Block Size"}
seen = set()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in want and d["Metric Name"] not in seen:
        seen.add(d["Metric Name"])
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ia, isrc, iss, iex = (hdr.index(x) for x in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                             "Instructions Executed"))
uniq = {}
for r in data:
    uniq.setdefault(r[ia], r)
data = list(uniq.values())
tot = {c: sum(int(r[hdr.index(c)] or 0) for r in data) for c in cols}
allsamp = sum(int(r[iss] or 0) for r in data)
print("stall totals:", {k: v for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v})
print("total samples", allsamp, "executed warp-instr", sum(int(r[iex] or 0) for r in data))
for r in sorted(data, key=lambda r: -int(r[iss] or 0))[:ntop]:
    reasons = {c[6:]: r[hdr.index(c)] for c in cols if r[hdr.index(c)] not in ("0", "")}
    print(f"{r[iss]:>7} {r[iex]:>8} {r[ia][-5:]} {r[isrc][:70]:70s} {reasons}")
