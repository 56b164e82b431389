# config-1 attention shape (B=8, H=32 MHA, T~2.3K): split-count sweep
mkdir -p gpurun_out/r2
for s in 0 1 2 3 4 6 8; do timeout 120 python tools/prof_attend.py --batch 8 --kv 32 --rep 1 --ctx 2304 --iters 50 --graph --splits $s 2>&1 | tail -1; done
for s in 0 1 2 3 4 6 8; do timeout 120 python tools/prof_attend.py --batch 8 --kv 32 --rep 1 --ctx 2304 --iters 50 --graph --splits $s --append 2>&1 | tail -1; done
