RP_LIB=ab/new.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -2
for i in 1 2; do
for L in base new; do
echo -n "$L: "; RP_LIB=ab/$L.so timeout 120 python tools/attn_window_one.py 64 197 16 104 --time
echo -n "$L: "; RP_LIB=ab/$L.so timeout 120 python tools/attn_window_one.py 64 512 12 64 --time
done; done
