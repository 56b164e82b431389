for v in base nofuse base nofuse; do
  if [ $v = base ]; then L=""; else L="OTT_LIB_PATH=tools/variants/$v.so"; fi
  echo "== $v"; env $L timeout 900 python bench.py --no-cpu --no-e2e --steps 16 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['avg_launch_us'], d['clocks']['sm_mhz'])"
done > gpurun_out/var.log 2>&1
