# bench line + launch list + ncu of the attention kernel (each ncu only after its plain run exits 0)
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$? >> gpurun_out/bench.err
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attend|flush|ring_write|combine" -c 800 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 2 > gpurun_out/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 1 -c 1 -o gpurun_out/mma_v8 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 2 > gpurun_out/ncu.log 2>&1
