RP_LIB=ab/new.so timeout 1200 python -m pytest tests/test_gpu_optim_stats.py tests/test_gpu_engine.py -q -x 2>&1 | tail -2
for P in revvit-g48 revvit-b; do
for L in base new base new; do
echo -n "$P $L: "; RP_LIB=ab/$L.so python tools/ab_step.py --preset $P --rounds 1 --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v['ms'],2) for k,v in d.items() if 'pdl0' in k})"
done; done
