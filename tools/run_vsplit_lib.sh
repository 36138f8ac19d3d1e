# ring-flush quant_kernel / flush_tc durations for library variants (tools/_var/<name>) x KVLC_VSPLIT values
#   tools/run_vsplit_lib.sh "base qk4" "2 4"
for v in $1; do for vs in $2; do
  if [ "$v" = base ]; then L=""; else L="tools/_var/$v/libkvlinc.so"; fi
  KVLC_LIB=$L KVLC_VSPLIT=$vs timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quant_kernel|flush_tc" --csv \
    --log-file gpurun_out/vsl.csv python tools/flushstep_launches.py > /dev/null 2>&1
  python - "$v" "$vs" <<'PY'
import csv, io, sys
t = open("gpurun_out/vsl.csv").read()
rows = list(csv.DictReader(io.StringIO(t[t.index('"ID"'):])))
print(sys.argv[1], "vsplit", sys.argv[2], [(r["Grid Size"], round(float(r["Metric Value"]) / 1e3, 1)) for r in rows])
PY
done; done
