timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --reps 2
python tools/prof_flush.py --batch 64 --kv 8 --ctx 4096 --reps 3
python tools/prof_flush.py --batch 64 --kv 8 --ctx 4096 --pool 3 --reps 3
ncu --set full --clock-control none --import-source on -k regex:flush_frozen -c 1 -o gpurun_out/frozen_v2 python tools/prof_flush.py --batch 64 --kv 8 --ctx 4096 --reps 1 > gpurun_out/ncu_frozen.log 2>&1
