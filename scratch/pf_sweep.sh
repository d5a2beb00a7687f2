for PF in 0 1 2 3 4 6; do
  LA_PREFETCH=$PF timeout 100 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pf_$PF.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pf_$PF.json')); print($PF, round(d['ms_per_step'],3), {k: round(v['ms'],3) for k,v in d['kernels'].items()})"
  LA_PREFETCH=$PF timeout 200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:"k_fwd_tc|k_bwd_tc" -s 2 -c 2 --csv python scratch/prof_fwd.py 65536 2>/dev/null | grep -E "dram__bytes|duration" | awk -F'","' '{print $5, $13, $14, $15}' | cut -c1-200
done
