for P in revvit-g48 rev-swin-b; do
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_list_$P.csv python tools/profile_step.py --preset $P --mode reprop > /dev/null 2>&1; echo ncu rc=$?
python tools/launch_table.py gpurun_out/s3_list_$P.csv > gpurun_out/s3_list_$P.md 2>&1; head -22 gpurun_out/s3_list_$P.md
done
