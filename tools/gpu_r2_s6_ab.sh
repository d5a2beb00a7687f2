# A/B of the in-sweep W_hat (default lib) against the staged W_hat (scratch/lib_staged.so):
# bitwise output hashes, backward parity tests, interleaved per-kernel times
set -u
mkdir -p gpurun_out
for L in paper_2510_21956_b200/libla_cuda.so scratch/lib_staged.so; do
  LA_CUDA_LIB=$PWD/$L timeout 300 python scratch/bitwise_libs.py > gpurun_out/s6_hash_$(basename $L).txt 2>&1; echo hash_rc=$?
done
diff gpurun_out/s6_hash_libla_cuda.so.txt gpurun_out/s6_hash_lib_staged.so.txt && echo BITWISE_SAME
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_geometry.py tests/test_dist.py tests/test_sharding.py -q -m gpu -p no:cacheprovider -x > gpurun_out/s6_ab_pytest.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/s6_ab_pytest.log
timeout 600 bash scratch/ab_libs.sh paper_2510_21956_b200/libla_cuda.so scratch/lib_staged.so > gpurun_out/s6_ab_times.txt 2>&1; echo ab_rc=$?
cat gpurun_out/s6_ab_times.txt
