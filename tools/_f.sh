mkdir -p gpurun_out
(
for b in 2 4 8; do
  python tools/prof_attend.py --batch 16 --kv 8 --rep 4 --ctx 4096 --iters 50 --graph --bits $b 2>&1 | tail -1
  python tools/prof_attend.py --batch 64 --kv 8 --rep 4 --ctx 8192 --iters 30 --graph --bits $b 2>&1 | tail -1
  python tools/prof_attend.py --batch 8 --kv 32 --rep 1 --ctx 2304 --iters 50 --graph --bits $b 2>&1 | tail -1
  python tools/prof_attend.py --batch 4 --kv 32 --rep 1 --ctx 32768 --iters 20 --graph --bits $b 2>&1 | tail -1
  python tools/prof_attend.py --batch 128 --kv 8 --rep 8 --ctx 16384 --iters 10 --graph --bits $b 2>&1 | tail -1
done
) > gpurun_out/sweep_bits.log 2>&1
cat gpurun_out/sweep_bits.log
