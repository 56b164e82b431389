# small-shape K2 probe (config 3: B=16, H_kv=8, n_rep=4, T=4096): split sweep + ncu launch times
mkdir -p gpurun_out/r2
O=gpurun_out/r2/small.log; : > $O
P="python tools/prof_attend.py --batch 16 --rep 4 --ctx 4096 --iters 50 --graph"
for s in 0 1 2 3 4 6 8; do timeout 120 $P --splits $s >> $O 2>&1; done
timeout 120 python tools/prof_attend.py --batch 64 --rep 4 --ctx 8192 --iters 50 --graph >> $O 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:"attend|combine" -c 10 --csv \
  python tools/prof_attend.py --batch 16 --rep 4 --ctx 4096 --iters 3 > gpurun_out/r2/small_ncu.csv 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 3 -c 1 -o gpurun_out/r2/ncu_small \
  python tools/prof_attend.py --batch 16 --rep 4 --ctx 4096 --iters 3 > gpurun_out/r2/ncu_small.log 2>&1
