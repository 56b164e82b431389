# api tests + default bench line + launch list; $1 = tag
mkdir -p gpurun_out/r2
T=${1:-x}
timeout 600 python -m pytest tests/test_gpu_api.py -q > gpurun_out/r2/api_$T.log 2>&1; echo "pytest_exit=$?" >> gpurun_out/r2/api_$T.log
timeout 1200 python bench.py > gpurun_out/r2/bench_$T.json 2> gpurun_out/r2/bench_$T.err; echo "bench_exit=$?" >> gpurun_out/r2/bench_$T.err
