#!/bin/bash
# A/B on one box: bench.py with scratch/ab/libla_cuda_base.so vs the current build, interleaved
# (extra args are passed as env assignments for the current build, e.g. LA_SEGMENTS=2)
for i in 1 2; do
  for L in scratch/ab/libla_cuda_base.so paper_2510_21956_b200/libla_cuda.so; do
    echo -n "$(basename $L) "
    LA_CUDA_LIB=$PWD/$L python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v['ms'],3) for k,v in d['kernels'].items()})"
  done
done
echo -n "current LA_SEGMENTS=2 "
LA_SEGMENTS=2 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v['ms'],3) for k,v in d['kernels'].items()})"
