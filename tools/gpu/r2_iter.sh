# quick iteration: parity subset, timing of both K2 kernels, ncu of the tcq kernel; $1 = tag
mkdir -p gpurun_out/r2
T=${1:-x}; O=gpurun_out/r2/iter_$T.log
: > $O
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "gqa or golden" >> $O 2>&1; echo "pytest_exit=$?" >> $O
for k in ${KERNELS:-tcq}; do
  OTT_ATTN_KERNEL=$k timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph >> $O 2>&1
done
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_tcq -s 1 -c 1 -o gpurun_out/r2/ncu_$T \
  python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 2 > gpurun_out/r2/ncu_${T}.log 2>&1
echo ncu_exit=$? >> $O
fi
