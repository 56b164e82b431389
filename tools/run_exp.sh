timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
for v in base nopdl base nopdl; do
  if [ $v = base ]; then L=""; else L="OTT_LIB_PATH=tools/variants/$v.so"; fi
  echo "== $v"
  for cfg in "16 8 4 4096" "64 8 4 8192" "128 8 8 16384" "8 32 1 2304"; do set -- $cfg
    env $L timeout 120 python tools/prof_attend.py --batch $1 --kv $2 --rep $3 --ctx $4 --iters 50 --graph 2>&1 | tail -1; done
  env $L timeout 300 python tools/prof_c1.py --steps 16 2>&1 | tail -1
done > gpurun_out/var.log 2>&1
