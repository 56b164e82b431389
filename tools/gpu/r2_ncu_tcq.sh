# ncu --set full of one attention launch (config-4 layer); $1 = tag, $2 = kernel regex, env passes OTT_ATTN_KERNEL
mkdir -p gpurun_out/r2
T=${1:-tcq}; K=${2:-attend_tcq}
timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 3 > gpurun_out/r2/ncu_${T}_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/r2/ncu_$T \
  python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 2 > gpurun_out/r2/ncu_${T}.log 2>&1
echo exit=$? >> gpurun_out/r2/ncu_${T}.log
