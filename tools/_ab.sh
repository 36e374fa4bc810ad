timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k gemm 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm python -m paper_2306_09342_b200.ncu_targets 2>&1 | grep -E "gemm_sm100|duration" | sed -e 's/(CUtensorMap.*//' | paste - - | awk '{print $2, $NF}' | tail -7
