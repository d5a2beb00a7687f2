# non-causal tcgen05 kernels (la_full.cu): parity tests first, then the config-4 geometry
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -k "noncausal or unaligned or small_and_edge or head_dim" -x > gpurun_out/pytest_full.log 2>&1; echo full_rc=$?
tail -30 gpurun_out/pytest_full.log
rm -f gpurun_out/parity_full.jsonl
LA_PARITY_LOG=gpurun_out/parity_full.jsonl timeout 900 python -m pytest tests/test_parity_geometry.py -q -m gpu -p no:cacheprovider -k config4 > gpurun_out/pytest_full_geom.log 2>&1; echo geom_rc=$?
tail -5 gpurun_out/pytest_full_geom.log; cut -c1-300 gpurun_out/parity_full.jsonl
