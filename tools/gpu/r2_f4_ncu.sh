mkdir -p gpurun_out/r2
for lib in old:tools/variants/old_flush.so new:paper_2505_10938_b200/_lib/libott_b200.so; do
 n=${lib%%:*}; p=${lib#*:}
 OTT_LIB_PATH=$p timeout 600 ncu --set full --clock-control none --import-source on -k regex:flush_frozen4 -c 1 -o gpurun_out/r2/f4_$n -f python tools/prof_flush.py --batch 16 --kv 8 --ctx 16384 --pool 32 --bits 4 --reps 1 > gpurun_out/r2/f4_ncu_$n.log 2>&1
done
