#!/bin/bash
# One GPU call's worth of profiling for the round summaries under profiles/:
#   1. the launch list of the bench command (cold-cache, serialised per-launch times)
#   2. one `ncu --set full` capture of each tcgen05 kernel of the north-star step
# Usage (on the GPU box): bash tools/profile_round.sh <tag>   -> gpurun_out/<tag>_*.{csv,ncu-rep}
set -u
TAG=${1:-prof}
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/${TAG}_launches.csv $BENCH > $OUT/${TAG}_launches.log 2>&1
for K in k_bwd_tc k_fwd_tc k_bwd_aggR_tc k_fwd_agg_tc; do
  ncu --set full --clock-control none --import-source on -k "${K}" -s 3 -c 1 \
      -o $OUT/${TAG}_${K} -f $BENCH > $OUT/${TAG}_${K}.log 2>&1
done
