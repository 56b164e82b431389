bash tools/run_var2.sh prev base prev base
ncu --metrics gpu__time_duration.sum -k regex:combine --csv python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 3 --append 2>/dev/null | grep combine | awk -F'","' '{print $NF}' | head -3
