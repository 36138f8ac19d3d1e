"""Warp-stall samples per CUDA source line (ncu --import-source report, -lineinfo build).

usage: python tools/ncu_stalls.py REPORT [TOP]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = hdr = None
samples, reasons, text = collections.Counter(), collections.defaultdict(collections.Counter), {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].strip():
        continue
    key = (cur, r[0])
    text[key] = r[1].strip()[:70]
    try:
        samples[key] += int(float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0))
    except ValueError:
        continue
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                reasons[key][h[6:]] += int(float(r[i] or 0))
            except ValueError:
                pass
tot = sum(samples.values()) or 1
print(f"total samples {tot}")
for key, n in samples.most_common(top):
    rs = ", ".join(f"{k} {v * 100 // max(n, 1)}%" for k, v in reasons[key].most_common(3) if v)
    print(f"{n * 100.0 / tot:5.1f}% {key[0][:15]:15s}:{key[1]:>4s} {text[key]:70s} [{rs}]")
