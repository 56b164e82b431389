timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 > gpurun_out/var.log 2>&1
