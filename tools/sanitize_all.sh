set -x
O=gpurun_out/r02s; mkdir -p $O
timeout 600 python tools/sanitize_run.py > $O/plain.log 2>&1; echo plain=$?
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_run.py > $O/memcheck.log 2>&1; echo memcheck=$?
timeout 1500 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_run.py > $O/synccheck.log 2>&1; echo synccheck=$?
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 50 python tools/sanitize_run.py > $O/racecheck.log 2>&1; echo racecheck=$?
timeout 600 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_c1.json 2>$O/bench_c1.err; echo c1=$?
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2>$O/bench_c3.err; echo c3=$?
tail -5 $O/*.log
