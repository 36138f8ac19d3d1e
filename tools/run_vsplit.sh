# quant_kernel duration of the ring flush (config-2 flushing step) per KVLC_VSPLIT (ncu, serialised)
for vs in "$@"; do
  KVLC_VSPLIT=$vs timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quant_kernel|flush_tc" --csv \
    --log-file gpurun_out/vs_$vs.csv python tools/flushstep_launches.py > /dev/null 2>&1
  python - "$vs" <<'PY'
import csv, io, sys
t = open(f"gpurun_out/vs_{sys.argv[1]}.csv").read()
rows = list(csv.DictReader(io.StringIO(t[t.index('"ID"'):])))
print("vsplit", sys.argv[1], [(r["Kernel Name"][:20], r["Grid Size"], round(float(r["Metric Value"]) / 1e3, 1)) for r in rows])
PY
done
