timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python bench.py > gpurun_out/bench_v11.jsonl 2> gpurun_out/bench_v11.err; tail -1 gpurun_out/bench_v11.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['prefill'], d['clocks'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v11.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_bench_v11.log 2>&1; tail -2 gpurun_out/ncu_bench_v11.log
