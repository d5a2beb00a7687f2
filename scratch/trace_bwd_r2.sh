# run the backward-sweep timeline against the traced side library built by:
#   bash scratch/build_var.sh scratch/libla_trace.so la_sm100_bwd -DLA_TRACE -DLA_TRACE_G=5
LA_CUDA_LIB=scratch/libla_trace.so python scratch/trace_bwd_r2.py
