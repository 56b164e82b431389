mkdir -p gpurun_out/r2
O=gpurun_out/r2/timeline5.log; : > $O
export OTT_LIB_PATH=tools/variants/tl.so
for a in "--batch 16 --rep 8 --ctx 16384" "--batch 4 --kv 32 --rep 1 --ctx 32768" "--batch 74 --rep 8 --ctx 16384 --splits 1"; do
  timeout 300 python tools/prof_timeline.py $a >> $O 2>&1
done
