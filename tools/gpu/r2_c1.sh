# full GPU tests + config-1 bench line (throughput + fidelity); $1 = tag
mkdir -p gpurun_out/r2
T=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_$T.log 2>&1; echo "pytest_exit=$?" >> gpurun_out/r2/pytest_$T.log
timeout 1500 python bench.py --config c1 > gpurun_out/r2/c1_$T.json 2> gpurun_out/r2/c1_$T.err; echo "exit=$?" >> gpurun_out/r2/c1_$T.err
