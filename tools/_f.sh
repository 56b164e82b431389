timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > gpurun_out/bench_v13.jsonl 2> gpurun_out/bench_v13.err; tail -1 gpurun_out/bench_v13.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d['prefill']['ms_per_layer'], d['cpu_baseline']['value'], d['clocks'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v13_all.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_bench_v13.log 2>&1; grep -c "" gpurun_out/launches_v13_all.csv
