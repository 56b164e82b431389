# K1b prefill iteration: GPU tests, config-4 prefill timing, decode-flush launch list; $1 = tag
mkdir -p gpurun_out/r2
T=${1:-x}; O=gpurun_out/r2/flush3_$T.log; : > $O
timeout 900 python -m pytest tests -m gpu -x -q >> $O 2>&1; echo "pytest_exit=$?" >> $O
for n in 32 3; do timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool $n >> $O 2>&1; done
timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 32 --bits 4 >> $O 2>&1
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flush_frozen_kernel -s 1 -c 1 -o gpurun_out/r2/ncu_frozen_$T \
  python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 32 --reps 1 > gpurun_out/r2/ncu_frozen_$T.log 2>&1
echo ncu_exit=$? >> $O
fi
if [ -n "$FLUSHLIST" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^flush_kernel" -c 200 --csv \
  --log-file gpurun_out/r2/launches_decode_flush.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2/ncu_flushlist.log 2>&1
echo flushlist_exit=$? >> $O
fi
