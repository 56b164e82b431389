# full GPU test suite + config-4 attention timing (+ optional ncu of attend_mma); $1 = tag
mkdir -p gpurun_out/r2
T=${1:-x}; O=gpurun_out/r2/full_$T.log
: > $O
timeout 900 python -m pytest tests -m gpu -x -q >> $O 2>&1; echo "pytest_exit=$?" >> $O
timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph >> $O 2>&1
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 1 -c 1 -o gpurun_out/r2/ncu_$T \
  python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 2 > gpurun_out/r2/ncu_${T}.log 2>&1
echo ncu_exit=$? >> $O
fi
