mkdir -p gpurun_out/r2
T=${1:-x}
timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_parity.py -q -k "model or outlier_tracking or lossless or graph or decode" > gpurun_out/r2/model_$T.log 2>&1; echo "exit=$?" >> gpurun_out/r2/model_$T.log
timeout 1500 python bench.py --config c1 > gpurun_out/r2/c1_$T.json 2> gpurun_out/r2/c1_$T.err; echo "exit=$?" >> gpurun_out/r2/c1_$T.err
