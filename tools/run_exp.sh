timeout 300 python tools/prof_c1.py --steps 16 > gpurun_out/c1.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "decoder or device_counter" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
