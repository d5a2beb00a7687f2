# session-6 re-entry check: smoke, full GPU suite, north-star bench line
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6_smoke.log 2>&1; echo smoke_rc=$?
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/s6_pytest_gpu.log 2>&1; echo gpu_rc=$?
tail -3 gpurun_out/s6_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/s6_bench.log 2>&1; echo bench_rc=$?
tail -c 1500 gpurun_out/s6_bench.log
