#!/bin/bash
# A/B of the 3D stored-face ring apply on C5: prefetch depth (SKC_APPLY_FD)
for fd in 2 3 1; do
  echo -n "fd=$fd: "
  SKC_APPLY_FD=$fd python bench.py --config C5 --no-secondary --steps 1 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']['apply']; print(d['value'], round(k['ms']*1000/k['launches'],1), 'us/apply', round(k['gbs']), 'GB/s')"
done
