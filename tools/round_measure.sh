#!/bin/bash
# Round-end measurement on one GPU: bench line, ncu launch list + full captures,
# compute-sanitizer over every tcgen05 / fused / prologue kernel. Outputs in gpurun_out/.
set -u
TAG=${1:-r01s3}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1
python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c3.log 2>&1
python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_c5.log 2>&1
python tools/config_sweep.py > gpurun_out/${TAG}_configs.jsonl 2> gpurun_out/${TAG}_configs.err
bash tools/profile_round.sh $TAG
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T --kernel-regex kns=_tc --kernel-regex kns=fused \
    python tools/sanitize_run.py > gpurun_out/${TAG}_san_${T}.log 2>&1
done
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/${TAG}_san_memcheck_all.log 2>&1
tail -c 400 gpurun_out/${TAG}_bench.log; for f in gpurun_out/${TAG}_san_*.log; do echo "$f: $(tail -2 $f | tr '\n' ' ')"; done
