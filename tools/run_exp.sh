timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo exit=$? >> gpurun_out/bench_c1.err
