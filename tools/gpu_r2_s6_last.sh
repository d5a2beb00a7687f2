# last verification of the session: full GPU suite, smoke, config-4 D=128 line
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/l_smoke.log 2>&1; echo smoke_rc=$?
rm -f gpurun_out/l_parity_geometry.jsonl
LA_PARITY_LOG=gpurun_out/l_parity_geometry.jsonl timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/l_pytest_gpu.log 2>&1; echo gpu_rc=$?
tail -3 gpurun_out/l_pytest_gpu.log
timeout 300 python bench.py --config 4 --dim 128 --steps 10 --warmup 3 > gpurun_out/l_bench_c4_d128.log 2>&1; echo c4_rc=$?
tail -c 300 gpurun_out/l_bench_c4_d128.log
