#!/bin/bash
for PF in 0 1 2 4; do
  echo -n "PF=$PF "
  LA_PREFETCH=$PF python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v['ms'],3) for k,v in d['kernels'].items()})"
done
