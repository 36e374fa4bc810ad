timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -x > gpurun_out/s2_gelu_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s2_gelu_tests.log
tools/ab_multi.sh tools/gemm_epi_ab.py 2 ab/base.so ab/new.so
