# per-GPU shard of config 4 at N = 2 / 4 / 8 (B = 64 / 32 / 16 of the 128 sequences), split sweep
mkdir -p gpurun_out/r2
O=gpurun_out/r2/shard.log; : > $O
for b in 64 32 16; do
  for s in 0 2 3 4 5 6 8; do
    timeout 120 python tools/prof_attend.py --batch $b --rep 8 --ctx 16384 --iters 20 --graph --splits $s >> $O 2>&1
  done
done
