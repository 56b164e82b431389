mkdir -p gpurun_out/r2
O=gpurun_out/r2/timeline4.log; : > $O
P="python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph"
for s in 1 2 3 4 6 8; do timeout 120 $P --splits $s >> $O 2>&1; done
for s in 1 2 4; do OTT_LIB_PATH=tools/variants/tl.so timeout 300 python tools/prof_timeline.py --batch 128 --rep 8 --ctx 16384 --splits $s >> $O 2>&1; done
