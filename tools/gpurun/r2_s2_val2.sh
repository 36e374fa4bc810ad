timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/s2_val2_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s2_val2_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s2_val2_bench.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/s2_val2_bench.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['reprop']['value'], d['mfu'], d['e2e']['value'], d['revvit_l'], d['clocks'], d['roofline']['frac'])"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_val2_launches.csv python tools/profile_step.py --mode reprop > gpurun_out/s2_val2_prof.log 2>&1; echo ncu rc=$?
python tools/launch_table.py gpurun_out/s2_val2_launches.csv > gpurun_out/s2_val2_launches.md 2>&1; head -22 gpurun_out/s2_val2_launches.md
