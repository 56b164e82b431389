mkdir -p gpurun_out/r2
O=gpurun_out/r2/sub.log; : > $O
timeout 900 python -m pytest tests -m gpu -x -q >> $O 2>&1; echo "pytest_exit=$?" >> $O
for G in 32 64 128; do
for a in "--batch 128 --rep 8 --ctx 16384" "--batch 64 --rep 4 --ctx 8192" "--batch 8 --kv 32 --rep 1 --ctx 4096"; do
  echo "new: $(timeout 120 python tools/prof_attend.py $a --group $G --iters 20 --graph 2>&1 | tail -1)" >> $O
  echo "old: $(OTT_LIB_PATH=tools/variants/presub.so timeout 120 python tools/prof_attend.py $a --group $G --iters 20 --graph 2>&1 | tail -1)" >> $O
done; done
