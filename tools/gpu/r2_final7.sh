# closing evidence (final state: + decode flush on the split kernels): GPU tests, smoke, prefill timings,
# ncu of the 2-bit frozen kernel, bench c4 + reference arm + c1, bench launch list
mkdir -p gpurun_out/r2l
O=gpurun_out/r2l
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest_exit=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for b in 2 3 4; do timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 32 --bits $b >> $O/prefill.log 2>&1; done
timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 3 >> $O/prefill.log 2>&1
timeout 300 python tools/prof_flush.py --batch 16 --kv 8 --ctx 32768 --pool 3 >> $O/prefill.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flush_frozen_kernel -s 1 -c 1 -o $O/ncu_frozen \
  python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 32 --reps 1 > $O/ncu_frozen.log 2>&1
timeout 1200 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "exit=$?" >> $O/bench_c4.err
timeout 600 python bench.py --impl reference --steps 4 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 1500 python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"flush|attend_mma|combine|ring_write" -c 2000 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > $O/ncu_launch.log 2>&1
