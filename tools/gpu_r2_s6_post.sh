# after the D = 128 routing change: full GPU suite, config-4 lines, north-star line
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p_smoke.log 2>&1; echo smoke_rc=$?
rm -f gpurun_out/p_parity_geometry.jsonl
LA_PARITY_LOG=gpurun_out/p_parity_geometry.jsonl timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/p_pytest_gpu.log 2>&1; echo gpu_rc=$?
tail -3 gpurun_out/p_pytest_gpu.log
for D in 64 128 256; do timeout 300 python bench.py --config 4 --dim $D --steps 10 --warmup 3 > gpurun_out/p_bench_c4_d$D.log 2>&1; echo c4_d${D}_rc=$?; done
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/p_bench.log 2>&1; echo bench_rc=$?
timeout 900 python tools/config_sweep.py > gpurun_out/p_configs.jsonl 2> gpurun_out/p_configs.err; echo sweep_rc=$?
