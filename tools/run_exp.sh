bash tools/run_var.sh base q16smb5 q16s mb5 base q16smb5 > gpurun_out/var.log 2>&1
