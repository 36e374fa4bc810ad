timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention_fwd_bwd or impl_switch" > gpurun_out/s2_fb2_tests.log 2>&1; echo tests rc=$?
tail -4 gpurun_out/s2_fb2_tests.log
timeout 300 python tools/attn_bwd_ab.py 3 0 > gpurun_out/s2_fb2_ab.log 2>&1; echo ab rc=$?
cat gpurun_out/s2_fb2_ab.log | tail -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_fused -s 1 -c 1 -o gpurun_out/s2_fb2 python tools/attn_bwd_one.py 0 > gpurun_out/s2_fb2_ncu.log 2>&1; echo ncu rc=$?
