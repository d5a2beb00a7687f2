#!/bin/bash
for A in "" 1 2 4 8; do
  echo -n "A=${A:-auto} "
  LA_AGG_SPLIT=$A python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v['ms'],3) for k,v in d['kernels'].items()})"
done
