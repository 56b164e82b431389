# A/B of attend variants through the fused append_attend path: python ... per variant
for v in "$@"; do
  echo "== $v"
  if [ "$v" = base ]; then L=""; else L="OTT_LIB_PATH=tools/variants/$v.so"; fi
  env $L timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --append 2>&1 | tail -1
done
