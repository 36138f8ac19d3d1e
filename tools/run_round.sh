# round evidence: bench line (all configs), reference arm, ncu launch list + full captures
tag=${1:-r01b}
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -2 gpurun_out/bench_$tag.err
cat gpurun_out/bench_$tag.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2>&1; tail -1 gpurun_out/bench_ref_$tag.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"split_kernel|combine_kernel|stage_input" -s 20 -c 40 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 5 --warmup 3 --no-fa --no-cpu --no-extra > /dev/null 2>&1
[ -n "$FULL" ] && timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_kernel -s 6 -c 1 -o gpurun_out/split_$tag python bench.py --steps 3 --warmup 3 --no-fa --no-cpu --no-extra > gpurun_out/ncu_$tag.log 2>&1
tail -1 gpurun_out/ncu_$tag.log
