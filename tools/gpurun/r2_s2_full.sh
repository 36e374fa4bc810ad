timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/s2_full_tests.log 2>&1; echo tests rc=$?
tail -4 gpurun_out/s2_full_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s2_full_bench.log 2>&1; echo bench rc=$?
python - <<'PY'
import json
l=[x for x in open('gpurun_out/s2_full_bench.log') if x.startswith('{')][-1]; d=json.loads(l)
print(d['value'], d['reprop'], d['pareprop_gain_pct'], d['mfu'], d['e2e']['value'], d['clocks'])
PY
