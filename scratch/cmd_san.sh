CS=/usr/local/cuda/bin/compute-sanitizer
timeout -s KILL 900 $CS --tool memcheck python tools/sanitize_run.py --round2 > gpurun_out/san_mem.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/san_mem.log
timeout -s KILL 900 $CS --tool racecheck --racecheck-report hazard python tools/sanitize_run.py --round2 > gpurun_out/san_race.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/san_race.log
timeout -s KILL 900 $CS --tool synccheck python tools/sanitize_run.py --round2 > gpurun_out/san_sync.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/san_sync.log
timeout -s KILL 600 $CS --tool memcheck python tools/sanitize_run.py > gpurun_out/san_mem1.log 2>&1; echo "memcheck(r1 set) rc=$?"; tail -2 gpurun_out/san_mem1.log
