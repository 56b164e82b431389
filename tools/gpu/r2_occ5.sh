mkdir -p gpurun_out/r2
O=gpurun_out/r2/occ5.log; : > $O
for a in "--batch 16 --rep 8 --ctx 16384" "--batch 16 --rep 8 --ctx 16384 --splits 4" "--batch 32 --rep 8 --ctx 16384" "--batch 4 --kv 32 --rep 1 --ctx 32768" "--batch 16 --rep 4 --ctx 4096" "--batch 16 --rep 4 --ctx 4096 --splits 4" "--batch 64 --rep 4 --ctx 8192" "--batch 8 --kv 32 --rep 1 --ctx 2304" "--batch 128 --rep 8 --ctx 16384"; do
  echo "prod: $(timeout 120 python tools/prof_attend.py $a --iters 20 --graph 2>&1 | tail -1)" >> $O
  echo "occ5: $(OTT_LIB_PATH=tools/variants/occ5.so timeout 120 python tools/prof_attend.py $a --iters 20 --graph 2>&1 | tail -1)" >> $O
done
OTT_LIB_PATH=tools/variants/occ5.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> $O
