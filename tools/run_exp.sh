timeout 900 python -m pytest tests -m gpu -x -q -k "long_context" --durations=3 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
