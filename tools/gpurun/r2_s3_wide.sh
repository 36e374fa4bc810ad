timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "general_head_dim" 2>&1 | tail -3
python tools/attn_window_one.py 64 197 16 104 --time
python tools/attn_window_one.py 64 197 16 104 --time --impl=1
python tools/attn_window_one.py 64 197 16 104 --time
