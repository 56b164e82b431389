# bench line + launch list (each ncu only after its plain run exits 0)
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$? >> gpurun_out/bench.err
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attend|flush|ring_write|combine" -c 800 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 1500 python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
