nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/s2_val_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s2_val_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2_val_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/s2_val_bench.log 2>&1; echo bench rc=$?
tail -c 300 gpurun_out/s2_val_bench.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_val_launches.csv python tools/profile_step.py --mode reprop > gpurun_out/s2_val_prof.log 2>&1; echo ncu rc=$?
python tools/launch_table.py gpurun_out/s2_val_launches.csv > gpurun_out/s2_val_launches.md 2>&1; head -30 gpurun_out/s2_val_launches.md
