RP_LIB=ab/new.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "general_head_dim or attention_fwd_bwd" 2>&1 | tail -2
for i in 1 2; do
echo -n "base: "; RP_LIB=ab/base.so python tools/attn_window_one.py 64 197 16 104 --time
echo -n "new:  "; RP_LIB=ab/new.so python tools/attn_window_one.py 64 197 16 104 --time
done
