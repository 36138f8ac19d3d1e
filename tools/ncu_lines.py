"""Instructions executed per source line (ncu --import-source report, -lineinfo build)."""
import collections
import csv
import io
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, ix = None, None, None
by_line, text = collections.Counter(), {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ix = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= ix or not r[0].strip():
        continue
    try:
        n = int(r[ix] or 0)
    except ValueError:
        n = 0
    text[(cur, r[0])] = r[1].strip()[:78]
    by_line[(cur, r[0])] += n
tot = sum(by_line.values())
print(f"total {tot} ({tot / units:.0f} per unit)")
for (f, l), n in by_line.most_common(top):
    print(f"{n / units:7.1f} {f[:15]:15s}:{l:>4} {text.get((f, l), '')}")
