timeout 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_traffic.csv python tools/profile_step.py --mode reprop > gpurun_out/r2_traffic.log 2>&1; echo rc=$?
python tools/gemm_traffic.py gpurun_out/r2_traffic.csv gpurun_out/round2_gemm_traffic | head -40
