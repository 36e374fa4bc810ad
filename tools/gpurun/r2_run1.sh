set -x
nproc; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests/test_gpu_optim_stats.py tests/test_gpu_depth.py tests/test_gpu_dp.py -q -x -rs > gpurun_out/r2_newtests.log 2>&1; echo new rc=$?
timeout 900 python tests/depth_parity.py --out gpurun_out/r2_depth_parity > gpurun_out/r2_depth.log 2>&1; echo depth rc=$?
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/r2_gputests.log 2>&1; echo all rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench.log 2>&1; echo bench rc=$?
