# baseline check after container re-creation: gpu tests + bench line
tag=${1:-base}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -3 gpurun_out/bench_$tag.err
cat gpurun_out/bench_$tag.json
cat MEASURED_PEAKS.json 2>/dev/null; cp MEASURED_PEAKS.json gpurun_out/ 2>/dev/null
timeout 120 python tools/decode_probe.py perf 16 4 28 8192 0
timeout 120 python tools/decode_probe.py perf 1 8 32 131072 0
