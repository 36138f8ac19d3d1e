"""Writes profiles/split_kernel_traffic.json from an ncu --set full capture of split_kernel
(tools/run_ncu_dec.sh), tagged with the sha256 of the decode sources it was built from
(bench.py uses the traffic figure only while that hash matches).

    python tools/update_traffic.py gpurun_out/split_<tag>.ncu-rep <tag>
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import decode_source_hash  # noqa: E402

rep, tag = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
vals = rows[2] if len(rows) > 2 else rows[1]
units = rows[1]


def metric(name):
    i = hdr.index(name)
    v = float(vals[i].replace(",", ""))
    u = units[i].strip().lower()
    scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
    return v * scale.get(u, 1)


rd, wr = metric("dram__bytes_read.sum"), metric("dram__bytes_write.sum")
rec = {"dram_bytes_per_launch": int(rd + wr), "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
       "duration_us_cold_serialised": metric("gpu__time_duration.sum"),
       "capture": f"profiles/r02/ncu_split_kernel_{tag}_summary.txt", "source_sha256": decode_source_hash(),
       "how": "ncu --set full --clock-control none -k regex:split_kernel -s 6 -c 1, python bench.py "
              "--steps 3 --warmup 3 --no-fa --no-cpu --no-extra (config 2)"}
json.dump(rec, open(os.path.join(ROOT, "profiles", "split_kernel_traffic.json"), "w"), indent=1)
print(json.dumps(rec, indent=1))
