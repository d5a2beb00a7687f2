# round-2 session-3 first GPU call: full GPU suite, bench line, launch list + ncu captures
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
rm -f gpurun_out/parity_geometry.jsonl
LA_PARITY_LOG=gpurun_out/parity_geometry.jsonl timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo gpu_rc=$?
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo bench_rc=$?
timeout 900 bash tools/profile_round.sh r02s3 ; echo prof_rc=$?
tail -15 gpurun_out/pytest_gpu.log; cut -c1-200 gpurun_out/parity_geometry.jsonl; tail -c 1500 gpurun_out/bench_full.log
