timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "colsum or gemm_mul or layer_norm" 2>&1 | tail -3
tools/ab_multi.sh tools/colsum_ab.py 3 ab/base.so ab/new.so
tools/ab_multi.sh "tools/ab_step.py --rounds 1" 2 ab/base.so ab/new.so
