# chunks-per-split sweep of the default build: config 2 (bench) and config 4 / config 3 points
for r in 1 2; do for c in 0 8 12 16 20 24; do
  echo -n "cpc $c: "
  KVLC_CPC=$c python tools/ab_points.py 16:8:32:8192 1:8:32:131072 16:4:28:32768 2>&1 | tail -1
done; done
