timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100_2sm -s 7 -c 7 -o gpurun_out/s2_gemm_full python tools/ncu_targets.py > gpurun_out/s2_ncu_gemm.log 2>&1; echo rc=$?
tail -3 gpurun_out/s2_ncu_gemm.log
