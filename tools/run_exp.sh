timeout 600 python -m pytest tests -m gpu -x -q -k "ratio or trace" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
