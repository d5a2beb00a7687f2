timeout -s KILL 120 python scratch/fused_check.py 64 65536 20; echo "rc=$?"
timeout -s KILL 120 python scratch/tune_times.py bwd_fused=1; echo "rc=$?"
