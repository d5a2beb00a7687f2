# A/B: in-sweep W_hat with 8 / 1 / 2 / 16 units in flight, + dc on warps 2-3, against the staged W_hat
set -u
mkdir -p gpurun_out
timeout 900 bash scratch/ab_libs.sh paper_2510_21956_b200/libla_cuda.so scratch/lib_wb1.so scratch/lib_wb2.so scratch/lib_wb16.so scratch/lib_dcwg2.so scratch/lib_staged.so > gpurun_out/s6_ab2_times.txt 2>&1; echo ab_rc=$?
cat gpurun_out/s6_ab2_times.txt
