"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel: share, count, avg/min/max us."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
t = defaultdict(list)
for r in rows[1:]:
    if len(r) <= iv or r[iv] == "":
        continue
    v = float(r[iv].replace(",", ""))
    u = r[iu]
    v = v / 1e3 if u == "nsecond" else v * 1e3 if u == "msecond" else v if u == "usecond" else v / 1e3
    t[r[ik]].append(v)
tot = sum(sum(x) for x in t.values())
print(f"launch list ({sum(len(x) for x in t.values())} launches, {tot/1e3:.3f} ms total, cold-cache serialised)")
print(f"{'share':>7} {'n':>5} {'avg_us':>10} {'min_us':>9} {'max_us':>9}  kernel")
for k, x in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{100*sum(x)/tot:6.2f}% {len(x):5d} {sum(x)/len(x):10.1f} {min(x):9.1f} {max(x):9.1f}  {k[:80]}")
