# side library with one source recompiled with extra flags: build_var.sh <out.so> <src basename> <nvcc flags...>
set -e
cd "$(dirname "$0")/.."
out=$1; src=$2; shift 2
python -c "from paper_2510_21956_b200 import build as b; b.build()"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  "$@" -c paper_2510_21956_b200/csrc/$src.cu -o build/var_$src.o
objs=$(ls build/obj/*.o | grep -v "/$src.cu.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $objs build/var_$src.o -cudart shared -Xlinker -rpath=/usr/local/cuda/lib64
