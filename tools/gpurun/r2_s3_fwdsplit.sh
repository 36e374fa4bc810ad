timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "split_pv" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -3
timeout 300 python tools/attn_fwd_ab.py 3
timeout 120 python tools/attn_fwd_trace.py > gpurun_out/s3_fwd_trace.txt 2>&1; tail -3 gpurun_out/s3_fwd_trace.txt
