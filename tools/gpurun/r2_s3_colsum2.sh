timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "colsum" 2>&1 | tail -2
tools/ab_multi.sh tools/colsum_ab.py 2 ab/base.so ab/new.so
