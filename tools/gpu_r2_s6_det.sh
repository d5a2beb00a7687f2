# run-to-run determinism at config 4 (D = 64 / 128 / 256) and the north star; then a config-4 A/B
set -u
mkdir -p gpurun_out
for D in 64 128 256; do LA_CUDA_LIB=$PWD/scratch/lib_c4old.so timeout 300 python scratch/determinism_c4.py $D 30; done > gpurun_out/s6_det.txt 2>&1
LA_CUDA_LIB=$PWD/scratch/lib_c4old.so timeout 300 python scratch/determinism_c4.py 128 10 causal >> gpurun_out/s6_det.txt 2>&1
cat gpurun_out/s6_det.txt
DIMS="64 256" timeout 900 bash scratch/ab_c4g.sh scratch/lib_c4old.so scratch/lib_c4new.so > gpurun_out/s6_c4ab.txt 2>&1; cat gpurun_out/s6_c4ab.txt
