timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
bash tools/run_var2.sh prev base prev base
