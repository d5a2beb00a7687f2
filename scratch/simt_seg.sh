#!/bin/bash
for R in 256 128 64 32; do
  echo -n "min_rows=$R "
  LA_SIMT_SEG_ROWS=$R python tools/config_sweep.py 2>/dev/null | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_fwd_bwd'])"
done
