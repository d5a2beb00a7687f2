#!/bin/bash
# fused vs separate backward schedule over segment counts (ms per fwd+bwd step, per-kernel ms)
for P in 9 12 18 5; do
  for F in 1 0; do
    echo -n "P=$P fused=$F "
    LA_SEGMENTS=$P LA_BWD_FUSED=$F timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['ms_per_step'],3), {k: round(v['ms'],3) for k,v in d['kernels'].items()})"
  done
done
