RP_LIB=ab/new.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" 2>&1 | tail -2
tools/ab_multi.sh tools/gemm_epi_ab.py 3 ab/base.so ab/new.so
tools/ab_multi.sh "tools/ab_step.py --rounds 1 --steps 8" 2 ab/base.so ab/new.so
