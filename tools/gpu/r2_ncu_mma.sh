# ncu --set full of one mma.sync K2 launch (config-4 layer); $1 = tag
mkdir -p gpurun_out/r2
T=${1:-mma}
OTT_ATTN_KERNEL=mma timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph > gpurun_out/r2/iter_$T.log 2>&1
OTT_ATTN_KERNEL=mma timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 1 -c 1 -o gpurun_out/r2/ncu_$T \
  python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 2 > gpurun_out/r2/ncu_${T}.log 2>&1
echo ncu_exit=$? >> gpurun_out/r2/iter_$T.log
