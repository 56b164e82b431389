timeout 300 python -m pytest tests -m gpu -x -q -k "decoder" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
