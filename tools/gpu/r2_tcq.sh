# new tcgen05 K2 (default) vs the mma.sync K2 (OTT_ATTN_KERNEL=mma): timing + parity
mkdir -p gpurun_out/r2
O=gpurun_out/r2/tcq_${1:-a}.log
: > $O
timeout 120 python tools/prof_attend.py --batch 4 --rep 8 --ctx 2048 --iters 3 >> $O 2>&1; echo "small_exit=$?" >> $O
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "gqa or golden" >> $O 2>&1; echo "pytest_exit=$?" >> $O
for k in mma tcq; do
  OTT_ATTN_KERNEL=$k timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 >> $O 2>&1
  OTT_ATTN_KERNEL=$k timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph >> $O 2>&1
done
