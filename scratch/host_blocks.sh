#!/bin/bash
for B in 16 32 64; do
  echo -n "blocks=$B "
  LA_HOST_BLOCKS=$B python bench.py --steps 3 --warmup 3 --e2e-steps 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['e2e']['ms_per_step'],2), round(d['e2e']['value']/1e6,3))"
done
