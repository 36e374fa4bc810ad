timeout 900 python tests/depth_parity.py --out gpurun_out/r2_depth_parity > gpurun_out/r2_depth.log 2>&1; echo depth rc=$?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2_gputests.log 2>&1; echo all rc=$?
tail -15 gpurun_out/r2_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
