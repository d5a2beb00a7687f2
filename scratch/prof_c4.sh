# ncu of the config-4 D=64 backward passes (r, dq)
BENCH="python bench.py --config 4 --dim 64 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 40 --csv --log-file gpurun_out/c4_64_metrics.csv $BENCH > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_full_totals|k_full_apply" -s 6 -c 4 -o gpurun_out/c4_64_bwd -f $BENCH > gpurun_out/c4_64_ncu.log 2>&1
echo done
