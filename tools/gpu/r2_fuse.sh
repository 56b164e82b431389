mkdir -p gpurun_out/r2
O=gpurun_out/r2/fuse.log; : > $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q >> $O 2>&1; echo "pytest_exit=$?" >> $O
for rep in 1 2; do
for a in "--batch 128 --rep 8 --ctx 16384" "--batch 96 --rep 8 --ctx 16384" "--batch 148 --rep 8 --ctx 16384"; do
  echo "new: $(timeout 120 python tools/prof_attend.py $a --iters 20 --graph 2>&1)" >> $O
  echo "old: $(OTT_LIB_PATH=tools/variants/tail3.so timeout 120 python tools/prof_attend.py $a --iters 20 --graph 2>&1)" >> $O
done; done
