timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -2
python tools/attn_window_one.py 64 512 12 64 --time
python tools/attn_window_one.py 64 197 16 104 --time
python tools/attn_window_one.py 64 300 12 64 --time
