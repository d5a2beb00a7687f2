set -u
mkdir -p gpurun_out
{ echo "== warfence"; LA_CUDA_LIB=$PWD/scratch/lib_warfence.so timeout 300 python scratch/determinism_c4.py 64 30 fwd 2>&1 | tail -2
  LA_CUDA_LIB=$PWD/scratch/lib_warfence.so timeout 300 python scratch/determinism_c4.py 64 20 2>&1 | tail -2
  DIMS="64" timeout 600 bash scratch/ab_c4g.sh scratch/lib_c4old.so scratch/lib_warfence.so; } > gpurun_out/s6_det6.txt 2>&1
cat gpurun_out/s6_det6.txt
