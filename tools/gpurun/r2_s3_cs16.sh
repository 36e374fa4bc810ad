RP_LIB=ab/new.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "colsum or layer_norm or gemm_gelu_slope" 2>&1 | tail -2
tools/ab_multi.sh tools/colsum_ab.py 2 ab/base.so ab/new.so
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_cs_new.csv env RP_LIB=ab/new.so python tools/profile_step.py --preset rev-swin-b --mode reprop > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_cs_base.csv env RP_LIB=ab/base.so python tools/profile_step.py --preset rev-swin-b --mode reprop > /dev/null 2>&1
for f in base new; do python tools/launch_table.py gpurun_out/s3_cs_$f.csv | grep -E "total|colsum"; done
