timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for v in base vsmem base vsmem; do
  if [ $v = base ]; then L=""; else L="OTT_LIB_PATH=tools/variants/$v.so"; fi
  echo "== $v"; env $L python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --reps 2
done
