timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
for cfg in "64 4 8192" "16 4 4096" "128 8 16384" "16 4 8192" "64 4 4096"; do set -- $cfg; timeout 120 python tools/prof_attend.py --batch $1 --rep $2 --ctx $3 --iters 30 2>&1 | tail -1; done > gpurun_out/splits.log 2>&1
timeout 300 python tools/prof_c1.py --steps 16 > gpurun_out/c1.log 2>&1
