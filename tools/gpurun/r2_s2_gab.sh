tools/ab_multi.sh tools/gemm_epi_ab.py 3 ab/base.so ab/new.so
RP_LIB=ab/new.so python tools/gemm_trace.py
