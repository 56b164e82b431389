# attention across the BASELINE shapes at 2/4/8 bits (graph replay, 50 launches)
mkdir -p gpurun_out/r2s
O=gpurun_out/r2s/sweep2.log; : > $O
for b in 2 4 8; do
for a in "--batch 16 --kv 8 --rep 4 --ctx 4096" "--batch 16 --kv 8 --rep 4 --ctx 8192" "--batch 64 --kv 8 --rep 4 --ctx 4096" \
         "--batch 64 --kv 8 --rep 4 --ctx 8192" "--batch 128 --kv 8 --rep 8 --ctx 16384" "--batch 8 --kv 32 --rep 1 --ctx 2304" \
         "--batch 4 --kv 32 --rep 1 --ctx 32768" "--batch 1 --kv 32 --rep 1 --ctx 1024"; do
  echo "bits=$b $(timeout 120 python tools/prof_attend.py $a --iters 50 --graph --bits $b 2>&1 | tail -1)" >> $O
done; done
