mkdir -p gpurun_out/r2
O=gpurun_out/r2/stream.log; : > $O
timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph >> $O 2>&1
OTT_LIB_PATH=tools/variants/stream.so timeout 120 python tools/prof_attend.py --batch 128 --rep 8 --ctx 16384 --iters 20 --graph >> $O 2>&1
timeout 120 python tools/prof_peer_wait.py >> $O 2>&1
