timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention_fwd_bwd or impl_switch" > gpurun_out/s2_fb3_tests.log 2>&1; echo tests rc=$?
tail -4 gpurun_out/s2_fb3_tests.log
timeout 300 python tools/attn_bwd_ab.py 3 0 > gpurun_out/s2_fb3_ab.log 2>&1; echo ab rc=$?
cat gpurun_out/s2_fb3_ab.log | tail -8
python tools/attn_bwd_trace.py 2>&1 | tail -16
