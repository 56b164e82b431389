ncu --set full --clock-control none --import-source on -k regex:attend_mma8 -s 1 -c 1 -o gpurun_out/mma8_v1 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 2 --bits 8 > gpurun_out/ncu_mma8.log 2>&1
tail -1 gpurun_out/ncu_mma8.log
