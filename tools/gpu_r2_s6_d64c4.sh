# non-causal D = 128 through la_full.cu (per-pass kernels) vs the fused k_fwd_full_tc / k_bwd_full_tc
set -u
mkdir -p gpurun_out
LA_CUDA_LIB=$PWD/scratch/lib_d64c4.so timeout 900 python -m pytest tests/test_parity_geometry.py tests/test_parity_gpu.py tests/test_abi.py -q -m gpu -p no:cacheprovider -x > gpurun_out/s6_d64c4_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/s6_d64c4_pytest.log
DIMS="64" timeout 600 bash scratch/ab_c4g.sh scratch/lib_base.so scratch/lib_d64c4.so > gpurun_out/s6_d64c4_ab.txt 2>&1; cat gpurun_out/s6_d64c4_ab.txt
