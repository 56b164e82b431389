# ncu of the prefill scan + score kernels at config 2 (N = 3: the pool keeps competing for every group)
mkdir -p gpurun_out/r2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"flush_scan|flush_score|flush_frozen" -c 3 -o gpurun_out/r2/ncu_scan3 -f \
  python tools/prof_flush.py --batch 16 --kv 8 --ctx 32768 --pool 3 --reps 1 > gpurun_out/r2/ncu_scan3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:flush_ --csv --log-file gpurun_out/r2/scan3_launches.csv \
  python tools/prof_flush.py --batch 16 --kv 8 --ctx 32768 --pool 3 --reps 1 > /dev/null 2>&1
