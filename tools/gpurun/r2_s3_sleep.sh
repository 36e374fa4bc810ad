RP_LIB=ab/new.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -2
for i in 1 2; do
for L in base new; do
echo -n "$L: "; RP_LIB=ab/$L.so python tools/attn_window_one.py 256 197 12 64 --time
echo -n "$L: "; RP_LIB=ab/$L.so python tools/attn_window_one.py 64 512 12 64 --time
done; done
tools/ab_multi.sh "tools/gemm_epi_ab.py" 2 ab/base.so ab/new.so
tools/ab_multi.sh "tools/ab_step.py --rounds 1 --steps 5" 2 ab/base.so ab/new.so
