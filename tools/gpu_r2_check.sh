set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
LA_PARITY_LOG=gpurun_out/parity_geometry.jsonl timeout 900 python -m pytest tests/test_parity_geometry.py -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_geom.log 2>&1; echo geom_rc=$?
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench1.log 2>&1; echo bench_rc=$?
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider --deselect tests/test_parity_geometry.py > gpurun_out/pytest_gpu.log 2>&1; echo gpu_rc=$?
tail -3 gpurun_out/pytest_gpu.log; tail -5 gpurun_out/pytest_geom.log; tail -c 3000 gpurun_out/bench1.log
