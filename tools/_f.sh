mkdir -p gpurun_out
python bench.py > gpurun_out/bench_v10.jsonl 2> gpurun_out/bench_v10.err; tail -1 gpurun_out/bench_v10.jsonl | head -c 3500
