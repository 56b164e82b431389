# tail schedule A/B: GPU tests, config-4 layer at splits 2 (tail schedule) vs 1; $1 = tag
mkdir -p gpurun_out/r2
T=${1:-x}; O=gpurun_out/r2/tail_$T.log; : > $O
timeout 900 python -m pytest tests -m gpu -x -q >> $O 2>&1; echo "pytest_exit=$?" >> $O
P="python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph"
for r in 1 2; do for s in 0 1 4; do timeout 120 $P --splits $s >> $O 2>&1; done; done
timeout 120 python tools/prof_attend.py --batch 148 --rep 8 --ctx 16384 --iters 20 --graph >> $O 2>&1
timeout 120 python tools/prof_attend.py --batch 96 --rep 8 --ctx 16384 --iters 20 --graph >> $O 2>&1
