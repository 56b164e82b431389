# how much does the split combine cost in the step? (variant: combine launch skipped, timing only)
mkdir -p gpurun_out/r2
for i in 1 2; do
 for nc in 0 1; do
  if [ $nc = 1 ]; then E="OTT_LIB_PATH=tools/variants/nocomb.so OTT_NOCOMBINE=1"; else E=""; fi
  echo "nocombine=$nc"; env $E timeout 300 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph 2>&1 | tail -1
  env $E timeout 900 python bench.py --steps 16 --warmup 3 --no-e2e --no-cpu --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
 done
done
