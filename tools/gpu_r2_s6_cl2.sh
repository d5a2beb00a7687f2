# A/B: backward sweep as 2-CTA clusters (the two segments of a group co-scheduled) vs plain grid
set -u
mkdir -p gpurun_out
for L in scratch/lib_base.so scratch/lib_cl2.so; do
  LA_CUDA_LIB=$PWD/$L timeout 300 python scratch/bitwise_libs.py > gpurun_out/s6_hash_$(basename $L).txt 2>&1; echo hash_rc=$?
done
diff gpurun_out/s6_hash_lib_base.so.txt gpurun_out/s6_hash_lib_cl2.so.txt && echo BITWISE_SAME
timeout 600 bash scratch/ab_libs.sh scratch/lib_base.so scratch/lib_cl2.so > gpurun_out/s6_cl2_ab.txt 2>&1; cat gpurun_out/s6_cl2_ab.txt
