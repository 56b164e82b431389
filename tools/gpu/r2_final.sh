# final round-2 evidence: GPU tests, bench line (c4), c1 line, ncu of K2, bench launch list, peer wait
mkdir -p gpurun_out/r2f
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2f/pytest.log 2>&1; echo "pytest_exit=$?" >> gpurun_out/r2f/pytest.log
timeout 1200 python bench.py > gpurun_out/r2f/bench_c4.json 2> gpurun_out/r2f/bench_c4.err; echo "exit=$?" >> gpurun_out/r2f/bench_c4.err
timeout 600 python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/r2f/bench_ref.json 2> gpurun_out/r2f/bench_ref.err
timeout 1500 python bench.py --config c1 > gpurun_out/r2f/bench_c1.json 2> gpurun_out/r2f/bench_c1.err
timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph > gpurun_out/r2f/attend.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 1 -c 1 -o gpurun_out/r2f/ncu_attend \
  python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 2 > gpurun_out/r2f/ncu_attend.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2f/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^flush_kernel|attend_mma|combine|ring_write" -c 2000 --csv \
  --log-file gpurun_out/r2f/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2f/ncu_launch.log 2>&1
timeout 120 python tools/prof_peer_wait.py > gpurun_out/r2f/peer_wait.log 2>&1
