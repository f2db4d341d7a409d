"""Per-SASS-instruction breakdown of an ncu report (executed warp instructions, stall samples).
   python tools/ncu_sass.py rep.ncu-rep [n_top] [--by exec|stall]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 40
by = "stall" if "--by" in sys.argv and sys.argv[sys.argv.index("--by") + 1] == "stall" else "exec"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
recs = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        ex = int(d.get("Warp Instructions Executed", d.get("Instructions Executed", "0")) or 0)
        ss = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    recs.append((d["Address"], d["Source"].strip()[:80], ex, ss))
tot = sum(r[2] for r in recs)
tss = sum(r[3] for r in recs)
print(f"instructions {len(recs)}, executed warp-instr {tot}, stall samples {tss}")
# opcode histogram (executed)
ops = {}
for a, s, ex, ss in recs:
    op = s.split()[0] if s else "?"
    if op.startswith("@"):
        op = s.split()[1]
    op = op.split(".")[0]
    e = ops.get(op, (0, 0))
    ops[op] = (e[0] + ex, e[1] + ss)
print("# opcode  executed  share  stalls")
for op, (ex, ss) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"  {op:10s} {ex:10d} {100.0 * ex / max(tot, 1):5.1f}% {ss:6d}")
key = 3 if by == "stall" else 2
print(f"# top instructions by {by}")
for a, s, ex, ss in sorted(recs, key=lambda r: -r[key])[:ntop]:
    print(f"  {a:>6s} {ex:9d} {ss:5d}  {s}")
