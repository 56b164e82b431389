# how much does the split combine cost in the step? (variant: combine launch skipped, timing only)
# variant: ott_attend.cu with `if (getenv("OTT_NOCOMBINE")) return cudaSuccess;` at the top of launch_combine<D>,
# built by tools/build_variant.sh nocomb "" <that copy> into tools/variants/nocomb.so
mkdir -p gpurun_out/r2
for i in 1 2; do
 for nc in 0 1; do
  if [ $nc = 1 ]; then E="OTT_LIB_PATH=tools/variants/nocomb.so OTT_NOCOMBINE=1"; else E=""; fi
  echo "nocombine=$nc"; env $E timeout 300 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph 2>&1 | tail -1
  env $E timeout 900 python bench.py --steps 16 --warmup 3 --no-e2e --no-cpu --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
 done
done
