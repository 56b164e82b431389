# multirank test + compute-sanitizer racecheck / synccheck / memcheck of a small decode workload
mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_multirank.py -q > gpurun_out/r2/multirank.log 2>&1; echo "exit=$?" >> gpurun_out/r2/multirank.log
for t in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_step.py > gpurun_out/r2/sanitize_$t.log 2>&1
  echo "exit=$?" >> gpurun_out/r2/sanitize_$t.log
done
compute-sanitizer --version >> gpurun_out/r2/sanitize_racecheck.log 2>&1
