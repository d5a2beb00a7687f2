for pf in 0 1 2 4; do echo "PF=$pf"; PF=$pf LA_CUDA_LIB=scratch/libla_trace.so python scratch/trace_bwd_r2.py | grep -E "period|role 0 ev 4|role 3 ev 3|role 0 ev 2"; done
python scratch/pf_bwd.py 0 1 2 4 0
