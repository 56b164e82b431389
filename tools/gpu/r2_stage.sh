# frozen-kernel staging A/B (old = previous commit) + GPU suite
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do for lib in tools/variants/old_flush.so paper_2505_10938_b200/_lib/libott_b200.so; do
  for b in 2 4; do echo "$lib bits=$b"; OTT_LIB_PATH=$lib timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 32 --bits $b --reps 5; done; done; done
