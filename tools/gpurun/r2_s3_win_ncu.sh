python tools/attn_window_one.py --time
python tools/attn_window_one.py 8192 49 4 32 --time
python tools/attn_window_one.py 2048 49 8 32 --time
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_small|attn_bwd_dkdv|attn_bwd_dq" -s 3 -c 3 -o gpurun_out/s3_win python tools/attn_window_one.py > gpurun_out/s3_win_ncu.log 2>&1; echo ncu rc=$?
