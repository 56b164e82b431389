timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --reps 2
python tools/prof_flush.py --batch 64 --kv 8 --ctx 4096 --reps 3
