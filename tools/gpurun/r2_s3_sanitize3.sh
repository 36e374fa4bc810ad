mkdir -p gpurun_out/san
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_kernels.py > gpurun_out/san/round2_kernels_racecheck.log 2>&1; echo racecheck rc=$?; tail -2 gpurun_out/san/round2_kernels_racecheck.log
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -2
python tools/attn_window_one.py 64 512 12 64 --time
