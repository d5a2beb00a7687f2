# A/B: backward-sweep register split (setmaxnreg) 96/136 (shipped) vs 96/128 vs 120/128
set -u
mkdir -p gpurun_out
for L in scratch/lib_base.so scratch/lib_r128.so scratch/lib_r120.so; do
  LA_CUDA_LIB=$PWD/$L timeout 300 python scratch/bitwise_libs.py > gpurun_out/s6_hash_$(basename $L).txt 2>&1; echo hash_rc=$?
done
diff gpurun_out/s6_hash_lib_base.so.txt gpurun_out/s6_hash_lib_r128.so.txt && diff gpurun_out/s6_hash_lib_base.so.txt gpurun_out/s6_hash_lib_r120.so.txt && echo BITWISE_SAME
timeout 600 bash scratch/ab_libs.sh scratch/lib_base.so scratch/lib_r128.so scratch/lib_r120.so > gpurun_out/s6_regs_ab.txt 2>&1; cat gpurun_out/s6_regs_ab.txt
