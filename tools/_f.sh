OTT_ERRLOG=gpurun_out/err4.log timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
for b in 2 4; do python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 10 --bits $b 2>&1 | tail -1; done
python tools/prof_attend.py --batch 64 --rep 4 --ctx 8192 --iters 10 --bits 4 2>&1 | tail -1
