mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2/smi.txt 2>&1
timeout 300 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 > gpurun_out/r2/base_attend.log 2>&1
timeout 300 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph >> gpurun_out/r2/base_attend.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/r2/pytest_gpu.log
