mkdir -p gpurun_out/r2
O=gpurun_out/r2/flush2.log; : > $O
for lib in "" "OTT_LIB_PATH=tools/variants/flush_pre.so"; do
  echo "== $lib" >> $O
  for a in "" "--pool 3"; do env $lib timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --reps 3 $a >> $O 2>&1; done
done
