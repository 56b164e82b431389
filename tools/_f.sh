OTT_ERRLOG=gpurun_out/err8.log timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for b in 8 4 2; do python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 10 --bits $b 2>&1 | tail -1; done
