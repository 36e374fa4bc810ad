python tools/attn_window_one.py 64 512 12 64 --time
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_tc_long|attn_bwd_tc" -s 3 -c 3 -o gpurun_out/s3_rob python tools/attn_window_one.py 64 512 12 64 > gpurun_out/s3_rob_ncu.log 2>&1; echo ncu rc=$?
