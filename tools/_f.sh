for v in prev base prev base; do
  if [ $v = base ]; then L=""; else L="OTT_LIB_PATH=tools/variants/$v.so"; fi
  env $L python bench.py --no-cpu > gpurun_out/bench_ab.jsonl 2> gpurun_out/bench_ab.err; echo "$v $(tail -1 gpurun_out/bench_ab.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), round(d['roofline']['avg_launch_us'],1), d['clocks']['sm_mhz'])")"
done
