timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/s3_val5_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s3_val5_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_val5_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/s3_val5_smoke.log
timeout 900 python bench.py > gpurun_out/s3_val5_bench.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/s3_val5_bench.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['reprop']['value'], d['mfu'], d['e2e']['value'], d.get('revvit_l',{}).get('pareprop_img_s'), d['clocks'], d['roofline']['frac'])"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_val5_launches.csv python tools/profile_step.py --mode reprop > gpurun_out/s3_val5_prof.log 2>&1; echo ncu rc=$?
python tools/launch_table.py gpurun_out/s3_val5_launches.csv > gpurun_out/s3_val5_launches.md 2>&1; head -14 gpurun_out/s3_val5_launches.md
timeout 1200 python -m paper_2306_09342_b200.cli bench configs/rev_roberta_base.cfg > gpurun_out/s3_val5_rob.log 2>&1; echo rob rc=$?; tail -4 gpurun_out/s3_val5_rob.log
