for c in revvit_g48 rev_roberta_base; do
timeout 1500 python -m paper_2306_09342_b200.cli bench configs/$c.cfg > gpurun_out/s3_cfg2_$c.log 2>&1; echo $c rc=$?; grep -v '^{' gpurun_out/s3_cfg2_$c.log | tail -10
done
