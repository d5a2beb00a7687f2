# D = 64 non-causal nondeterminism: forward only vs fwd+bwd, with and without chunk pairing
set -u
mkdir -p gpurun_out
for L in scratch/lib_c4old.so scratch/lib_nopair.so; do
  echo "== $L"
  LA_CUDA_LIB=$PWD/$L timeout 300 python scratch/determinism_c4.py 64 20 fwd 2>&1 | tail -4
  LA_CUDA_LIB=$PWD/$L timeout 300 python scratch/determinism_c4.py 64 20 2>&1 | tail -4
done > gpurun_out/s6_det2.txt 2>&1
cat gpurun_out/s6_det2.txt
