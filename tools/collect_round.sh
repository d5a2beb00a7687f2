# Copy one round-measurement call's outputs (tools/gpu_r2_s*_final.sh) from gpurun_out/ into
# profiles/ under a tag: collect_round.sh <tag> (e.g. r02_s6)
set -eu
T=$1
O=gpurun_out
tail -1 $O/f_bench.log > profiles/${T}_bench.json
tail -1 $O/f_bench_ref.log > profiles/${T}_bench_reference.json
for C in 3 5; do tail -1 $O/f_bench_c$C.log > profiles/${T}_bench_c$C.json; done
for D in 64 128 256; do tail -1 $O/f_bench_c4_d$D.log > profiles/${T}_bench_c4_d$D.json; done
cp $O/f_configs.jsonl profiles/${T}_configs.jsonl
cp $O/parity_geometry.jsonl profiles/${T}_parity_geometry.jsonl
tail -30 $O/f_pytest_gpu.log > profiles/${T}_pytest_gpu.txt
[ -f $O/f_ab_ns.txt ] && cp $O/f_ab_ns.txt profiles/${T}_ab_north_star.txt
TAG=$(echo $T | tr -d _)
cp $O/${TAG}_launches.csv profiles/${T}_launches.csv
{ echo "# ncu --set full of the north-star kernels ($T, 1x B200)"; echo
  echo "Same command as tools/profile_round.sh (bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline), one capture per kernel. The bench line of this box: profiles/${T}_bench.json."
  for K in k_fwd_agg_tc k_fwd_tc k_bwd_aggR_tc k_bwd_tc; do python tools/ncu_summary.py $O/${TAG}_$K.ncu-rep $K; done; } > profiles/${T}_ncu.md
