# one bench line + per-kernel times (quick A/B on the GPU box)
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1; echo bench_rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.log").read().strip().splitlines()[-1])
print(d["ms_per_step"], {k: round(v["ms"], 4) for k, v in d["kernels"].items()})
PY
