# fp-tier pipeline check: GPU tests + attention timings on config-4 / config-1 / config-3 / 4-bit shapes; $1 = tag
mkdir -p gpurun_out/r2
T=${1:-x}; O=gpurun_out/r2/fp_$T.log; : > $O
timeout 900 python -m pytest tests -m gpu -x -q >> $O 2>&1; echo "pytest_exit=$?" >> $O
for a in "--batch 128 --rep 8 --ctx 16384" "--batch 8 --kv 32 --rep 1 --ctx 2304" "--batch 16 --rep 4 --ctx 4096" "--batch 64 --rep 4 --ctx 8192" "--batch 128 --rep 8 --ctx 16384 --bits 4"; do
  timeout 120 python tools/prof_attend.py $a --iters 20 --graph >> $O 2>&1
done
