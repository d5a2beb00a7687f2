for i in 1 2; do for L in "$@"; do
  for gn in "16 4096" "64 65536" "16 131072" "8 4096"; do LA_CUDA_LIB=$PWD/$L python scratch/kern_times.py $gn; done
done; done
