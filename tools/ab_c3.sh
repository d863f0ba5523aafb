for rep in 1 2; do
for d in ab_old .; do
  (cd $d && python bench.py --config C3s4 --no-secondary --steps 3 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$d', d['value'], {k:(round(v['ms']),v['gbs']) for k,v in d['kernels'].items() if v['ms']>5})")
done; done
