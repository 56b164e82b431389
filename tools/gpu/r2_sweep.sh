# attention across the BASELINE shapes (graph replay) + decode-flush launch list + frozen-kernel ncu
mkdir -p gpurun_out/r2s
O=gpurun_out/r2s/sweep.log; : > $O
for a in "--batch 16 --kv 8 --rep 4 --ctx 4096" "--batch 16 --kv 8 --rep 4 --ctx 8192" "--batch 64 --kv 8 --rep 4 --ctx 4096" \
         "--batch 64 --kv 8 --rep 4 --ctx 8192" "--batch 128 --kv 8 --rep 8 --ctx 16384" "--batch 8 --kv 32 --rep 1 --ctx 2300" \
         "--batch 4 --kv 32 --rep 1 --ctx 32768" "--batch 1 --kv 32 --rep 1 --ctx 1024"; do
  timeout 120 python tools/prof_attend.py $a --iters 50 --graph >> $O 2>&1
done
for b in 4 8; do timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph --bits $b >> $O 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attend|flush|ring_write|combine" -s 5600 -c 480 --csv \
  --log-file gpurun_out/r2s/launches_window.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2s/ncu_window.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flush_frozen_kernel -s 1 -c 1 -o gpurun_out/r2s/ncu_frozen \
  python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --reps 1 > gpurun_out/r2s/ncu_frozen.log 2>&1
timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --reps 3 > gpurun_out/r2s/flush.log 2>&1
