# config-4 launch lists with DRAM bytes (D = 64, 128, 256), one step after warm-up
for D in 64 128 256; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 60 --csv --log-file gpurun_out/c4_${D}_launches.csv python bench.py --config 4 --dim $D --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
echo done
