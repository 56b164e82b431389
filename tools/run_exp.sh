timeout 300 python -m pytest tests -m gpu -x -q -k "pipeline or smoke" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
bash tools/run_var.sh base mb3 mb5 st3 > gpurun_out/var.log 2>&1
for s in 1 3 4 6; do timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 10 --splits $s >> gpurun_out/var.log 2>&1; done
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
