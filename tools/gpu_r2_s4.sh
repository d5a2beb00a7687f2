# session-4 baseline: full GPU suite, smoke, bench lines (configs 2-5), launch list + ncu captures
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1; echo smoke_rc=$?
rm -f gpurun_out/parity_geometry.jsonl
LA_PARITY_LOG=gpurun_out/parity_geometry.jsonl timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s4_pytest_gpu.log 2>&1; echo gpu_rc=$?
tail -15 gpurun_out/s4_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/s4_bench.log 2>&1; echo bench_rc=$?
for C in 3 4 5; do timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4_bench_c$C.log 2>&1; echo c${C}_rc=$?; done
timeout 900 bash tools/profile_round.sh r02s4 ; echo prof_rc=$?
tail -c 1500 gpurun_out/s4_bench.log
