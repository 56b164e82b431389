# 3/4-bit frozen-pool flush A/B (old = tools/variants/old_flush.so) + the flush parity subset
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "bit_widths or adversarial or ties or generic_shapes or large_groups or any_query or golden" 2>&1 | tail -3
for b in 4 3 2; do
 for lib in tools/variants/old_flush.so paper_2505_10938_b200/_lib/libott_b200.so; do
  echo "$lib bits=$b"; OTT_LIB_PATH=$lib timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 32 --bits $b --reps 3
 done
done
OTT_LIB_PATH=paper_2505_10938_b200/_lib/libott_b200.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:flush_frozen4 -c 1 -o gpurun_out/r2/f4_new4 -f python tools/prof_flush.py --batch 16 --kv 8 --ctx 16384 --pool 32 --bits 4 --reps 1 > gpurun_out/r2/f4_ncu_new3.log 2>&1
