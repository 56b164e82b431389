mkdir -p gpurun_out/r2
T=${1:-x}; O=gpurun_out/r2/flush_$T.log; : > $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_cases.py tests/test_gpu_canary.py -q -x >> $O 2>&1; echo "pytest_exit=$?" >> $O
for a in "" "--pool 3" "--bits 4"; do timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --reps 3 $a >> $O 2>&1; done
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flush_frozen_kernel -s 1 -c 1 -o gpurun_out/r2/ncu_frozen_$T \
  python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --reps 1 > gpurun_out/r2/ncu_frozen_$T.log 2>&1
fi
