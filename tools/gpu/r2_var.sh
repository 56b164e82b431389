# time the product K2 and variants (tools/variants/<name>.so) on the config-4 layer; $@ = variant names
mkdir -p gpurun_out/r2
O=gpurun_out/r2/var_$(echo "$@" | tr ' ' '_').log; : > $O
P="python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph"
for rep in 1 2; do
  echo "== product" >> $O; timeout 120 $P >> $O 2>&1
  for v in "$@"; do echo "== $v" >> $O; OTT_LIB_PATH=tools/variants/$v.so timeout 120 $P >> $O 2>&1; done
done
for v in "$@"; do
  echo "== parity $v" >> $O
  OTT_LIB_PATH=tools/variants/$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2 >> $O
done
