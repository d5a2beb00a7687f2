# session-3 check: E_S split (WG-B / WG-C), workspace-only padded paths, la_sharded_* entry points
set -x
timeout 900 python -m pytest tests/test_dist.py tests/test_sharding.py tests/test_abi.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_dist.log 2>&1; echo dist_rc=$?
tail -15 gpurun_out/pytest_dist.log
rm -f gpurun_out/parity_geometry.jsonl
LA_PARITY_LOG=gpurun_out/parity_geometry.jsonl timeout 900 python -m pytest tests/test_parity_geometry.py -q -m gpu -p no:cacheprovider -k "config2 or config5" > gpurun_out/pytest_geom.log 2>&1; echo geom_rc=$?
tail -3 gpurun_out/pytest_geom.log; cut -c1-250 gpurun_out/parity_geometry.jsonl
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_par.log 2>&1; echo par_rc=$?
tail -3 gpurun_out/pytest_par.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1; echo bench_rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.log").read().strip().splitlines()[-1])
print(d["ms_per_step"], {k: round(v["ms"], 4) for k, v in d["kernels"].items()}, d["clocks"])
PY
bash scratch/trace_bwd_r2.sh > gpurun_out/trace_bwd.log 2>&1; tail -16 gpurun_out/trace_bwd.log
