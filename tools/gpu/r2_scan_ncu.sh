# ncu of the prefill scan kernel (config-4 layer, N = 32)
mkdir -p gpurun_out/r2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flush_scan -c 1 -o gpurun_out/r2/ncu_scan -f \
  python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 32 --reps 1 > gpurun_out/r2/ncu_scan.log 2>&1
