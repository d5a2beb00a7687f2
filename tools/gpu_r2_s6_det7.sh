set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_geometry.py -k "bitwise" -q -m gpu -p no:cacheprovider > gpurun_out/s6_det7.log 2>&1; echo rc=$?
tail -5 gpurun_out/s6_det7.log
