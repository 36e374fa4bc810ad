timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_g48_launches.csv python tools/profile_step.py --preset revvit-g48 --mode reprop > gpurun_out/s3_g48_prof.log 2>&1; echo ncu rc=$?
python tools/launch_table.py gpurun_out/s3_g48_launches.csv > gpurun_out/s3_g48_launches.md 2>&1; head -24 gpurun_out/s3_g48_launches.md
