timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s2_cfgs_bench.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/s2_cfgs_bench.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['reprop']['value'], d['revvit_l'], d['clocks'])"
for c in revvit_l rev_roberta_base revvit_g48 rev_swin_b; do
  timeout 900 python -m paper_2306_09342_b200.cli bench configs/$c.cfg --out gpurun_out/s2_cfg_$c.csv > gpurun_out/s2_cfg_$c.log 2>&1; echo $c rc=$?
  cat gpurun_out/s2_cfg_$c.csv
done
