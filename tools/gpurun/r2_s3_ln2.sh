RP_LIB=ab/new.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "layer_norm or colsum" 2>&1 | tail -2
tools/ab_multi.sh tools/ln_ab.py 2 ab/base.so ab/new.so
for L in base new base new; do
echo -n "swin $L: "; RP_LIB=ab/$L.so python tools/ab_step.py --preset rev-swin-b --rounds 1 --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v['ms'],2) for k,v in d.items() if 'pdl0' in k})"
done
