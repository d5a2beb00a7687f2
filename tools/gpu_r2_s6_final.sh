# session-6 round measurement: north-star A/B against the session-start library, full GPU
# suite, smoke, bench lines (ours + reference arm), config 3/4/5 lines, config sweep,
# launch list + ncu captures of the north-star kernels
set -u
mkdir -p gpurun_out
timeout 300 bash scratch/ab_libs.sh paper_2510_21956_b200/libla_cuda.so scratch/lib_c4old.so > gpurun_out/f_ab_ns.txt 2>&1; echo ab_rc=$?
cat gpurun_out/f_ab_ns.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke_rc=$?
rm -f gpurun_out/parity_geometry.jsonl
LA_PARITY_LOG=gpurun_out/parity_geometry.jsonl timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/f_pytest_gpu.log 2>&1; echo gpu_rc=$?
tail -3 gpurun_out/f_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/f_bench.log 2>&1; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_bench_ref.log 2>&1; echo ref_rc=$?
for C in 3 5; do timeout 600 python bench.py --config $C --steps 10 --warmup 3 > gpurun_out/f_bench_c$C.log 2>&1; echo c${C}_rc=$?; done
for D in 64 128 256; do timeout 300 python bench.py --config 4 --dim $D --steps 10 --warmup 3 > gpurun_out/f_bench_c4_d$D.log 2>&1; echo c4_d${D}_rc=$?; done
timeout 900 python tools/config_sweep.py > gpurun_out/f_configs.jsonl 2> gpurun_out/f_configs.err; echo sweep_rc=$?
timeout 1200 bash tools/profile_round.sh r02s6; echo prof_rc=$?
tail -c 600 gpurun_out/f_bench.log; echo; tail -c 400 gpurun_out/f_bench_ref.log
