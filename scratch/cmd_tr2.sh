for L in scratch/libla_trace.so scratch/libla_traceA.so; do echo "== $L"; LA_CUDA_LIB=$L python scratch/trace_bwd_r2.py | tail -23; done
