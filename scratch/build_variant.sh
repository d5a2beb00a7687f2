# side library with the pair kernel compiled with extra flags: build_variant.sh <out.so> <nvcc flags...>
set -e
cd "$(dirname "$0")/.."
out=$1; shift
python -c "from paper_2510_21956_b200 import build as b; b.build()"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  "$@" -c paper_2510_21956_b200/csrc/la_bwd_pair.cu -o build/pair_variant.o
objs=$(ls build/obj/*.o | grep -v la_bwd_pair)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $objs build/pair_variant.o -cudart shared -Xlinker -rpath=/usr/local/cuda/lib64
