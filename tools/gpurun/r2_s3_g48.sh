timeout 1200 python -m paper_2306_09342_b200.cli bench configs/revvit_g48.cfg > gpurun_out/s3_g48_bench.log 2>&1; echo rc=$?; tail -8 gpurun_out/s3_g48_bench.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_g48b_launches.csv python tools/profile_step.py --preset revvit-g48 --mode reprop > gpurun_out/s3_g48b_prof.log 2>&1; echo ncu rc=$?
python tools/launch_table.py gpurun_out/s3_g48b_launches.csv > gpurun_out/s3_g48b_launches.md 2>&1; head -16 gpurun_out/s3_g48b_launches.md
