"""Key metrics + stall reasons + SASS opcode mix from an ncu --set full report."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else None   # e.g. chunks per launch


def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
h, vals = raw[0], raw[2]
m = dict(zip(h, vals))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg"]
for k in keys:
    if k in m:
        print(f"{k:70s} {m[k]}")
stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for k, v in m.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and v.replace(".", "").isdigit()}
tot = sum(stalls.values()) or 1
print("stalls:", ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]))
src = page("source", ["--print-source", "sass"])
hh = src[1]
ix, isrc = hh.index("Instructions Executed"), hh.index("Source")
cnt = collections.Counter()
for r in src[2:]:
    if len(r) <= ix or not r[isrc].strip():
        continue
    toks = r[isrc].strip().split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    if not (r[ix] or "0").replace(",", "").isdigit():  # a repeated header (multi-kernel report)
        continue
    cnt[op.split(".")[0]] += int((r[ix] or "0").replace(",", ""))
total = sum(cnt.values())
div = units or 1
print(f"instructions {total} ({total / div:.0f} per unit)")
print("  ".join(f"{k}:{v / div:.0f}" for k, v in cnt.most_common(24)))
