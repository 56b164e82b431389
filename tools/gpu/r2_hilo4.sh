mkdir -p gpurun_out/r2
O=gpurun_out/r2/hilo4.log; : > $O
timeout 900 python -m pytest tests -m gpu -x -q >> $O 2>&1; echo "pytest_exit=$?" >> $O
for a in "--batch 16 --rep 4 --ctx 4096" "--batch 64 --rep 4 --ctx 8192" "--batch 8 --kv 32 --rep 1 --ctx 2304" "--batch 4 --kv 32 --rep 1 --ctx 32768" "--batch 128 --rep 8 --ctx 16384"; do
  echo "new: $(timeout 120 python tools/prof_attend.py $a --bits 4 --iters 20 --graph 2>&1 | tail -1)" >> $O
  echo "old: $(OTT_LIB_PATH=tools/variants/pre4.so timeout 120 python tools/prof_attend.py $a --bits 4 --iters 20 --graph 2>&1 | tail -1)" >> $O
done
