mkdir -p gpurun_out/r2
O=gpurun_out/r2/pick.log; : > $O
timeout 900 python -m pytest tests -m gpu -x -q >> $O 2>&1; echo "pytest_exit=$?" >> $O
for b in 128 64 32 16; do timeout 120 python tools/prof_attend.py --batch $b --rep 8 --ctx 16384 --iters 20 --graph >> $O 2>&1; done
for a in "--batch 16 --rep 4 --ctx 4096" "--batch 64 --rep 4 --ctx 8192" "--batch 8 --kv 32 --rep 1 --ctx 2304" "--batch 4 --kv 32 --rep 1 --ctx 32768"; do
  timeout 120 python tools/prof_attend.py $a --iters 20 --graph >> $O 2>&1; done
