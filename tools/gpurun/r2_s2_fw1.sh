timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" > gpurun_out/s2_fw1_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s2_fw1_tests.log
tools/ab_libs.sh tools/attn_time.py ab/base.so ab/new.so 3
python tools/attn_fwd_trace.py 2>&1 | tail -2
