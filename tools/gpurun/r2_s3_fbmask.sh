RP_LIB=ab/new.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -2
tools/ab_multi.sh "tools/attn_bwd_ab.py" 3 ab/base.so ab/new.so
