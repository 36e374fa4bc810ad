timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_rob_launches.csv python tools/profile_step.py --preset rev-roberta-base --mode reprop > gpurun_out/s3_rob_prof.log 2>&1; echo ncu rc=$?
python tools/launch_table.py gpurun_out/s3_rob_launches.csv > gpurun_out/s3_rob_launches.md 2>&1; head -16 gpurun_out/s3_rob_launches.md
