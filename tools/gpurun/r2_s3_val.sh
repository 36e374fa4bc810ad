timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/s3_val_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s3_val_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_val_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/s3_val_smoke.log
timeout 900 python bench.py > gpurun_out/s3_val_bench.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/s3_val_bench.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['reprop']['value'], d['mfu'], d['e2e']['value'], d.get('revvit_l'), d['clocks'], d['roofline']['frac'], d.get('cpu_baseline',{}).get('value'))"
timeout 900 python -m paper_2306_09342_b200.cli bench configs/rev_swin_b.cfg > gpurun_out/s3_val_swin.log 2>&1; echo swin rc=$?; tail -5 gpurun_out/s3_val_swin.log
