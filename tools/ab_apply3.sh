#!/bin/bash
# A/B of the 3D constant-stencil ring apply on C3s4: tile rows (SKC_APPLY_TY), prefetch depth
# (SKC_APPLY_D) and planes per CTA (SKC_APPLY_KZ; 0 = the wave-fitting choice)
for ty in 4 8; do for dd in 1 2 4; do for kz in 0 16; do
  echo -n "ty=$ty d=$dd kz=$kz: "
  SKC_APPLY_TY=$ty SKC_APPLY_D=$dd SKC_APPLY_KZ=$kz python bench.py --config C3s4 --no-secondary --steps 1 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']['apply']; print(d['value'], round(k['ms']*1000/k['launches'],1), 'us/apply', round(k['gbs']), 'GB/s')"
done; done; done
