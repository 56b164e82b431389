# final round-2 evidence (after the tail schedule and the prefill work)
mkdir -p gpurun_out/r2g
O=gpurun_out/r2g
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest_exit=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 1200 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "exit=$?" >> $O/bench_c4.err
timeout 600 python bench.py --impl reference --steps 4 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 1500 python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph > $O/attend.log 2>&1
timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 32 > $O/prefill.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 1 -c 1 -o $O/ncu_attend \
  python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 2 > $O/ncu_attend.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flush_frozen_kernel -s 1 -c 1 -o $O/ncu_frozen \
  python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 32 --reps 1 > $O/ncu_frozen.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attend_mma|combine|ring_write|flush_scan|flush_frozen" -c 1300 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^flush_kernel" -c 200 --csv \
  --log-file $O/launches_decode_flush.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > $O/ncu_flushlist.log 2>&1
