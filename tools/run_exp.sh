for cfg in "16 8 4 4096" "16 8 4 8192" "64 8 4 4096" "64 8 4 8192" "128 8 8 16384" "8 32 1 2304" "1 32 1 1024" "4 32 1 32768"; do
  set -- $cfg
  timeout 120 python tools/prof_attend.py --batch $1 --kv $2 --rep $3 --ctx $4 --iters 50 --graph 2>&1 | tail -1
done > gpurun_out/sweep.log 2>&1
