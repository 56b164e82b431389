timeout 1500 python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo exit=$? >> gpurun_out/bench_c1.err
