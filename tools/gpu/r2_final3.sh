mkdir -p gpurun_out/r2h
O=gpurun_out/r2h
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest_exit=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 1500 python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 1200 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "exit=$?" >> $O/bench_c4.err
