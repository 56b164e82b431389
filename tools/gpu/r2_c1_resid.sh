# config-1 decoder: residual adds fused into RMSNorm (beta = 0 GEMMs) vs the previous commit
# (tools/variants/prev = that commit's package with its library), + model/decoder tests, + bench c1
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_parity.py -x -q -m gpu -k "model or decoder or rmsnorm or rope or device_counter or flash or lossless or outlier_tracking" 2>&1 | tail -3
for i in 1 2; do
  echo prev; timeout 300 python tools/variants/prev/tools/prof_c1.py --steps 20 2>&1 | tail -1
  echo new; timeout 300 python tools/prof_c1.py --steps 20 2>&1 | tail -1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2/c1_launches3.csv python tools/prof_c1.py --steps 1 > /dev/null 2>&1
timeout 1500 python bench.py --config c1 > gpurun_out/r2/bench_c1_resid.json 2> gpurun_out/r2/bench_c1_resid.err
