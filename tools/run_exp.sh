timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
bash tools/run_var.sh base prev base prev > gpurun_out/var.log 2>&1
