timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
bash tools/run_var.sh base prev base prev > gpurun_out/var.log 2>&1
for v in base prev; do
  if [ $v = base ]; then L=""; else L="OTT_LIB_PATH=tools/variants/$v.so"; fi
  echo "== $v c3"; env $L timeout 120 python tools/prof_attend.py --batch 16 --rep 4 --ctx 4096 --iters 50 2>&1 | tail -1
done >> gpurun_out/var.log 2>&1
