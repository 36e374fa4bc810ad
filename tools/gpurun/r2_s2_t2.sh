./tools/umma_bench > gpurun_out/s2_umma.txt 2>&1; cat gpurun_out/s2_umma.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/s2_gputests2.log 2>&1; echo all rc=$?
tail -5 gpurun_out/s2_gputests2.log
