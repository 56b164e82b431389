mkdir -p gpurun_out/r2
O=gpurun_out/r2/tcq2_$1.log; : > $O
for s in 1 3; do
  echo "tcq: $(OTT_LIB_PATH=tools/variants/tcq.so timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph --splits $s 2>&1 | tail -1)" >> $O
done
echo "product: $(timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph 2>&1 | tail -1)" >> $O
OTT_LIB_PATH=tools/variants/tcq.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "attention or gqa or attend" 2>&1 | tail -2 >> $O
if [ -n "$NCU" ]; then
OTT_LIB_PATH=tools/variants/tcq.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_tcq -s 1 -c 1 -o gpurun_out/r2/ncu_tcq_$1 \
  python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 2 --splits 1 > gpurun_out/r2/ncu_tcq_$1.log 2>&1
fi
