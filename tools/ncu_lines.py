"""Per-source-line instructions executed and stall samples for one kernel of an ncu report.

usage: python tools/ncu_lines.py REPORT KERNEL_REGEX [TOP]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
cur = hdr = None
ins, smp, text = collections.Counter(), collections.Counter(), {}
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0].strip().isdigit():
        continue
    key = (cur, int(r[0]))
    text[key] = r[1].strip()[:72]
    try:
        ins[key] += float(r[7] or 0)
        smp[key] += float(r[4] or 0)
    except ValueError:
        pass
ti, ts = sum(ins.values()) or 1, sum(smp.values()) or 1
print(f"warp instructions {ti:.4g}, stall samples {ts:.4g}")
for k, v in ins.most_common(top):
    print(f"{100 * v / ti:5.1f}% inst {100 * smp[k] / ts:5.1f}% smp  {k[0][:15]:15s}:{k[1]:5d} {text[k]}")
