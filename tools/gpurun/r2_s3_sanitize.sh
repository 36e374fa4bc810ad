mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck; do
timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_kernels.py > gpurun_out/san/round2_kernels_$t.log 2>&1; echo $t rc=$?; tail -3 gpurun_out/san/round2_kernels_$t.log
done
