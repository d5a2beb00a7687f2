# Build a clock64-traced copy of the library (separate dir) and dump the backward sweep timeline.
set -e
OUT=/tmp/latrace; mkdir -p $OUT
for f in paper_2510_21956_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -DLA_TRACE -DLA_TRACE_G=${TG:-5} -c $f -o $OUT/$(basename $f).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libla_cuda.so $OUT/*.o -cudart shared
LA_CUDA_LIB=$OUT/libla_cuda.so python scratch/trace_bwd_r2.py
