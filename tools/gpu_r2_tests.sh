# full GPU suite + geometry parity log + one bench line
rm -f gpurun_out/parity_geometry.jsonl
LA_PARITY_LOG=gpurun_out/parity_geometry.jsonl timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo gpu_rc=$?
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo bench_rc=$?
tail -15 gpurun_out/pytest_gpu.log; cat gpurun_out/parity_geometry.jsonl | cut -c1-200; tail -c 400 gpurun_out/bench_full.log
