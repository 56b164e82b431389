# N = 3 prefill A/B (scan skip window kept in registers; old = previous commit) + GPU suite
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do for lib in tools/variants/old_flush.so paper_2505_10938_b200/_lib/libott_b200.so; do
  echo "$lib config2"; OTT_LIB_PATH=$lib timeout 300 python tools/prof_flush.py --batch 16 --kv 8 --ctx 32768 --pool 3 --reps 5
  echo "$lib c4 N=3"; OTT_LIB_PATH=$lib timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 3 --reps 3
done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:flush_ --csv --log-file gpurun_out/r2/window_launches.csv \
  python tools/prof_flush.py --batch 16 --kv 8 --ctx 32768 --pool 3 --reps 1 > /dev/null 2>&1
