nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/s2_gputests.log 2>&1; echo all rc=$?
tail -5 gpurun_out/s2_gputests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s2_bench.log 2>&1; echo bench rc=$?
tail -c 600 gpurun_out/s2_bench.log
