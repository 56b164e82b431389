# config-1 decoder elementwise kernels: numerics tests + A/B (old = previous commit's library) + launch list
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_model.py -x -q -m gpu 2>&1 | tail -3
for i in 1 2; do for lib in tools/variants/old_model.so paper_2505_10938_b200/_lib/libott_b200.so; do
  echo "$lib"; OTT_LIB_PATH=$lib timeout 300 python tools/prof_c1.py --steps 20 2>&1 | tail -1; done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2/c1_launches2.csv python tools/prof_c1.py --steps 1 > /dev/null 2>&1
