timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "window or general_head_dim" 2>&1 | tail -2
for v in 0 0; do
python tools/attn_window_one.py --time --variant=$v
python tools/attn_window_one.py 8192 49 4 32 --time --variant=$v
done
python tools/attn_window_one.py 2048 49 8 32 --time
python tools/attn_window_one.py 128 49 32 32 --time
