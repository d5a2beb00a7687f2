# round-2 check: headline-geometry parity (all checks logged) + one bench line
rm -f gpurun_out/parity_geometry.jsonl
LA_PARITY_LOG=gpurun_out/parity_geometry.jsonl timeout 1200 python -m pytest tests/test_parity_geometry.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_geom.log 2>&1; echo geom_rc=$?
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_geom.log 2>&1; echo bench_rc=$?
tail -5 gpurun_out/pytest_geom.log; cat gpurun_out/parity_geometry.jsonl; tail -c 600 gpurun_out/bench_geom.log
