mkdir -p gpurun_out/r2
O=gpurun_out/r2/fpab.log; : > $O
for rep in 1 2; do
for a in "--batch 128 --rep 8 --ctx 16384" "--batch 8 --kv 32 --rep 1 --ctx 2304" "--batch 16 --rep 4 --ctx 4096" "--batch 64 --rep 4 --ctx 8192" "--batch 128 --rep 8 --ctx 16384 --bits 4"; do
  echo "new: $(timeout 120 python tools/prof_attend.py $a --iters 20 --graph 2>&1)" >> $O
  echo "old: $(OTT_LIB_PATH=tools/variants/fpold.so timeout 120 python tools/prof_attend.py $a --iters 20 --graph 2>&1)" >> $O
done; done
