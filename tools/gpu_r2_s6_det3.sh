set -u
mkdir -p gpurun_out
LA_CUDA_LIB=$PWD/scratch/lib_c4old.so timeout 300 python scratch/det_probe_c4.py > gpurun_out/s6_det3.txt 2>&1
cat gpurun_out/s6_det3.txt
