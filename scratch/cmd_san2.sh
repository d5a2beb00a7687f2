CS=/usr/local/cuda/bin/compute-sanitizer
s=$(date +%s.%N); python tools/sanitize_run.py --round2 > /dev/null 2>&1; e=$(date +%s.%N); echo "plain $(python3 -c "print(round($e - $s, 2))")"
s=$(date +%s.%N); $CS --tool racecheck python tools/sanitize_run.py --round2 > gpurun_out/san_race2.log 2>&1; e=$(date +%s.%N); echo "racecheck $(python3 -c "print(round($e - $s, 2))")"; tail -1 gpurun_out/san_race2.log
s=$(date +%s.%N); $CS --tool racecheck --kernel-regex kns=k_full_apply python tools/sanitize_run.py --round2 > /dev/null 2>&1; e=$(date +%s.%N); echo "racecheck k_full_apply only $(python3 -c "print(round($e - $s, 2))")"
s=$(date +%s.%N); $CS --tool memcheck --launch-skip 100000 python tools/sanitize_run.py --round2 > /dev/null 2>&1; e=$(date +%s.%N); echo "memcheck none checked $(python3 -c "print(round($e - $s, 2))")"
s=$(date +%s.%N); $CS --tool memcheck python tools/sanitize_run.py --round2 > /dev/null 2>&1; e=$(date +%s.%N); echo "memcheck all $(python3 -c "print(round($e - $s, 2))")"
