timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
bash tools/run_var.sh base > gpurun_out/var.log 2>&1
timeout 120 python tools/prof_attend.py --batch 64 --rep 4 --ctx 8192 --iters 50 >> gpurun_out/var.log 2>&1
timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 2 > gpurun_out/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 1 -c 1 -o gpurun_out/mma_v7 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 2 > gpurun_out/ncu.log 2>&1
