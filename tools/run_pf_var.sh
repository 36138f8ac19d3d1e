# config-5 flush_tc_kernel / quant_kernel time per library variant (tools/_var/<name>), ncu serialised
for v in base "$@"; do
  if [ "$v" = base ]; then L=""; else L="tools/_var/$v/libkvlinc.so"; fi
  KVLC_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quant_kernel|flush_tc" -s 2 -c 2 --csv \
    --log-file gpurun_out/pfv.csv python tools/bench_prefill.py --steps 2 --warmup 1 > /dev/null 2>&1
  echo "$v: $(python tools/launch_summary.py gpurun_out/pfv.csv | tail -2 | awk '{print $1, $3}' | tr '\n' ' ')"
done
