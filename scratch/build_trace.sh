# traced pair kernel in a side library (the product library stays trace-free)
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2510_21956_b200 import build as b; b.build()"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  -DLA_TRACE -DLA_TRACE_W0=${W0:-256} -c paper_2510_21956_b200/csrc/la_bwd_pair.cu -o build/pair_trace.o
objs=$(ls build/obj/*.o | grep -v la_bwd_pair)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scratch/libla_trace.so $objs build/pair_trace.o -cudart shared -Xlinker -rpath=/usr/local/cuda/lib64
