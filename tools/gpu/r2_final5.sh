# closing evidence after the scan copy batching: GPU tests, smoke, prefill (2/3/4-bit, N=3), bench c4, launch list
mkdir -p gpurun_out/r2j
O=gpurun_out/r2j
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest_exit=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for b in 2 3 4; do timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 32 --bits $b >> $O/prefill.log 2>&1; done
timeout 300 python tools/prof_flush.py --batch 128 --kv 8 --ctx 16384 --pool 3 >> $O/prefill.log 2>&1
timeout 1200 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "exit=$?" >> $O/bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"flush|attend_mma|combine|ring_write" -c 2000 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > $O/ncu_launch.log 2>&1
