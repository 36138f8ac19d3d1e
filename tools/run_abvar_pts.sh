# interleaved same-box A/B of library variants (tools/_var/<name>) on decode points B:HKV:HQ:N
#   tools/run_abvar_pts.sh "v1 v2" "B:HKV:HQ:N ..."
for r in 1 2; do for v in base $1; do
  if [ "$v" = base ]; then L=""; else L="tools/_var/$v/libkvlinc.so"; fi
  echo -n "$v: "; KVLC_LIB=$L python tools/ab_points.py $2 2>&1 | tail -1
done; done
