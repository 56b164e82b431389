# frozen4 occupancy A/B: product (128 regs) vs min-blocks 5 / 6 builds
mkdir -p gpurun_out/r2
for lib in paper_2505_10938_b200/_lib/libott_b200.so tools/variants/f4_mb5.so tools/variants/f4_mb6.so; do
 for b in 4 3; do echo "$lib bits=$b"; OTT_LIB_PATH=$lib timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 32 --bits $b --reps 3; done
done
