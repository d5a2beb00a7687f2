for i in 1 2; do for L in "$@"; do for D in ${DIMS:-64 256}; do
  echo -n "$L D=$D "; LA_CUDA_LIB=$PWD/$L python bench.py --config 4 --dim $D --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v['ms'],3) for k,v in d.get('kernels',{}).items()})"
done; done; done
