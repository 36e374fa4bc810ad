./tools/tmem_mufu_bench > gpurun_out/r2_tmem_mufu.txt 2>&1; cat gpurun_out/r2_tmem_mufu.txt
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_reprop.csv python tools/profile_step.py --mode reprop > gpurun_out/r2_prof.log 2>&1; echo ncu rc=$?
python tools/launch_table.py gpurun_out/r2_launches_reprop.csv | head -40
