# session 4: pair-backward tests, non-causal rename check, config-4 bench lines, config sweep
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pair.py tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -x -k "pair or noncausal or head_dim" > gpurun_out/s4b_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/s4b_pytest.log
for D in 64 128 256; do timeout 300 python bench.py --config 4 --dim $D --steps 10 --warmup 3 > gpurun_out/s4b_bench_c4_d$D.log 2>&1; echo c4_d${D}_rc=$?; done
timeout 900 python tools/config_sweep.py > gpurun_out/s4b_configs.jsonl 2> gpurun_out/s4b_configs.err; echo sweep_rc=$?
python - <<'PY'
import json
for D in (64, 128, 256):
    try:
        d = json.loads(open(f"gpurun_out/s4b_bench_c4_d{D}.log").read().strip().splitlines()[-1])
        print(D, round(d["ms_per_step"], 4), {k: round(v["frac"], 3) for k, v in d["phases"].items()}, d["e2e"]["ms_per_step"] if d.get("e2e") else None)
    except Exception as e:
        print(D, "ERR", e)
PY
cut -c1-220 gpurun_out/s4b_configs.jsonl
