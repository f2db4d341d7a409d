"""Per-CUDA-source-line breakdown (executed warp instructions and stall samples) of an ncu report
captured with --import-source on and a -lineinfo build.
   python tools/ncu_lines.py gpurun_out/prof.ncu-rep [n_top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, agg = None, None, {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[0] == "":
        continue
    key = (cur, int(r[0]))
    ex, ss = int(r[7] or 0), int(r[4] or 0)
    o = agg.get(key, (0, 0, r[1].strip()[:95]))
    agg[key] = (o[0] + ex, o[1] + ss, o[2])
tot = sum(v[0] for v in agg.values())
tss = sum(v[1] for v in agg.values())
print(f"total executed warp-instr {tot}, stall samples {tss}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:ntop]:
    print(f"{v[0]:>9} {100.0 * v[0] / max(tot, 1):5.1f}% {v[1]:>6} {k[0][:14]:>14}:{k[1]:<5} {v[2]}")
