bash tools/run_var.sh base > gpurun_out/var.log 2>&1
timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 >> gpurun_out/var.log 2>&1
timeout 120 python tools/prof_attend.py --batch 64 --rep 4 --ctx 8192 --iters 50 >> gpurun_out/var.log 2>&1
