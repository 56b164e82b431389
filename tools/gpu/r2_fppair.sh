mkdir -p gpurun_out/r2
O=gpurun_out/r2/fppair.log; : > $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q >> $O 2>&1; echo "pytest_exit=$?" >> $O
for rep in 1 2; do
for a in "--batch 16 --splits 3" "--batch 16 --splits 4" "--batch 32 --splits 4" "--batch 64 --splits 2"; do
  echo "$(timeout 120 python tools/prof_attend.py --rep 8 --ctx 16384 --iters 20 --graph $a 2>&1 | tail -1)" >> $O
done; done
for a in "--batch 16 --rep 4 --ctx 4096 --splits 4" "--batch 16 --rep 4 --ctx 4096 --splits 3" "--batch 4 --kv 32 --rep 1 --ctx 32768 --splits 4"; do
  echo "$(timeout 120 python tools/prof_attend.py --iters 20 --graph $a 2>&1 | tail -1)" >> $O
done
