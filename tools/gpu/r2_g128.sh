mkdir -p gpurun_out/r2
O=gpurun_out/r2/g128.log; : > $O
for G in 32 64 128; do
  timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph --group $G >> $O 2>&1
  timeout 120 python tools/prof_attend.py --batch 64 --rep 4 --ctx 8192 --iters 20 --graph --group $G >> $O 2>&1
done
