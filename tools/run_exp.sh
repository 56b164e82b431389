timeout 900 python -m pytest tests -m gpu -x -q -k "golden or config0 or stress or bit_widths" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
for v in base fmb4 prev; do
  if [ $v = base ]; then L=""; else L="OTT_LIB_PATH=tools/variants/$v.so"; fi
  echo "== $v"; env $L timeout 120 python tools/prof_flush.py --batch 16 --kv 8 --ctx 4096 2>&1 | tail -1
  env $L timeout 120 python tools/prof_flush.py --batch 128 --kv 8 --ctx 4096 2>&1 | tail -1
  env $L timeout 120 python tools/prof_flush.py --batch 8 --kv 32 --ctx 2048 2>&1 | tail -1
done > gpurun_out/flush.log 2>&1
