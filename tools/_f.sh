timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --reps 2
python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 3 --reps 2
python tools/prof_flush.py --batch 4 --kv 32 --ctx 32768 --pool 3 --reps 2
python tools/prof_flush.py --batch 4 --kv 32 --ctx 32768 --pool 3 --reps 2 --bits 4
