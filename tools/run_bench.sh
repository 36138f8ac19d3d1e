# one GPU call: bench line, reference arm, ncu launch list + full capture of the split kernel
tag=${1:-r1}
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -3 gpurun_out/bench_$tag.err
cat gpurun_out/bench_$tag.json
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$tag.json 2>&1; cat gpurun_out/bench_ref_$tag.json | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 3 --warmup 3 --no-fa --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_kernel -s 6 -c 1 -o gpurun_out/split_$tag python bench.py --steps 3 --warmup 3 --no-fa --no-cpu > gpurun_out/ncu_$tag.log 2>&1
tail -2 gpurun_out/ncu_$tag.log
