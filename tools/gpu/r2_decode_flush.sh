# decode flushes through the scan + frozen kernels (old = previous commit: flush_kernel) + GPU suite
mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for lib in tools/variants/old_flush.so paper_2505_10938_b200/_lib/libott_b200.so tools/variants/old_flush.so paper_2505_10938_b200/_lib/libott_b200.so; do
  echo $lib; OTT_LIB_PATH=$lib timeout 900 python bench.py --steps 32 --warmup 3 --no-e2e --no-cpu --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['decode_flush'], d['clocks']['sm_mhz'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"flush" -c 400 --csv \
  --log-file gpurun_out/r2/decode_flush_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > /dev/null 2>&1
