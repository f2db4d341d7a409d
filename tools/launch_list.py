"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel name.
   python tools/launch_list.py launches.csv "header comment" > profiles/<name>.txt"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hd = rows[h]
ki, vi, ui = hd.index("Kernel Name"), hd.index("Metric Value"), hd.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] == "ns" else (v * 1e3 if r[ui] == "ms" else v)  # -> us
    name = r[ki].split("(")[0] if not r[ki].startswith("void ") else r[ki][5:].split("(")[0]
    tot[name] += v
    cnt[name] += 1
all_us = sum(tot.values())
if len(sys.argv) > 2:
    print("#", sys.argv[2])
print(f"# launches {sum(cnt.values())}, total {all_us / 1e3:.1f} ms")
for n, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{cnt[n]:6d} {v:10.1f} us {100 * v / all_us:5.1f}%  avg {v / cnt[n]:8.2f} us  {n}")
