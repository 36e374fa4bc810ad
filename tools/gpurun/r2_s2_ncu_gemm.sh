timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100_2sm -s 7 -c 7 -o gpurun_out/s2_gemm_full python -m paper_2306_09342_b200.ncu_targets > gpurun_out/s2_ncu_gemm.log 2>&1; echo rc=$?
tail -3 gpurun_out/s2_ncu_gemm.log
