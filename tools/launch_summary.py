"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.reader(lines))
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    if len(r) > iv:
        name = r[ik].split("(")[0].replace("void ", "").replace("kvlc::<unnamed>::", "")[:70]
        d[name].append(float(r[iv].replace(",", "")) / 1000)
tot = sum(sum(v) for v in d.values())
print(f"{'kernel':70s} {'n':>5s} {'mean us':>9s} {'total us':>10s} {'share':>6s}")
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:70s} {len(v):5d} {sum(v)/len(v):9.2f} {sum(v):10.1f} {sum(v)/tot*100:5.1f}%")
