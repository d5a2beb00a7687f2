set -u
mkdir -p gpurun_out
for L in scratch/lib_redown.so scratch/lib_nototpf.so; do
  echo "== $L"
  LA_CUDA_LIB=$PWD/$L timeout 300 python scratch/determinism_c4.py 64 20 fwd 2>&1 | tail -2
done > gpurun_out/s6_det5.txt 2>&1
cat gpurun_out/s6_det5.txt
