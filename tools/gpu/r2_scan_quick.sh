mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "golden or config or generic or pool or ties or adversarial" 2>&1 | tail -2
for i in 1 2; do for lib in tools/variants/old_flush.so paper_2505_10938_b200/_lib/libott_b200.so; do
  echo "$lib"; OTT_LIB_PATH=$lib timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 32 --reps 5; done; done
