timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_c1.py --steps 16 > gpurun_out/c1.log 2>&1
