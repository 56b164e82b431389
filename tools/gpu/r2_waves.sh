# wave-quantisation probe for K2: config-4 layer at split counts 1-4, and batches at whole waves
mkdir -p gpurun_out/r2
O=gpurun_out/r2/waves.log; : > $O
P="python tools/prof_attend.py --rep 8 --ctx 16384 --iters 20 --graph"
for s in 1 2 3 4 6; do timeout 120 $P --batch 128 --splits $s >> $O 2>&1; done
for b in 74 111 148; do timeout 120 $P --batch $b --splits 1 >> $O 2>&1; done
