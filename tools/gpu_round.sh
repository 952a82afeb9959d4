#!/bin/bash
# One gpurun session: GPU tests, smoke, a bench line, and the ncu launch list of the same
# bench command. Usage (from the repo root, on the GPU box):
#   bash tools/gpu_round.sh TAG [tests|bench|ncu|full]...
# Writes everything under gpurun_out/TAG/.
TAG=${1:-run}; shift
STAGES=${@:-tests bench ncu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/gpu.txt 2>&1
for st in $STAGES; do
  case $st in
    tests)
      timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/rc.txt ;;
    bench)
      timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt ;;
    benchq)
      timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt ;;
    ref)
      timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?" >> $OUT/rc.txt ;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
        --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile-phases 0 \
        > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/rc.txt ;;
    full)
      # one --set full capture of each top kernel (by name regex in $KREGEX), source-mapped
      timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-raster_bwd}" -s ${KSKIP:-40} -c ${KCOUNT:-1} \
        -o $OUT/full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile-phases 0 \
        > $OUT/ncu_full.log 2>&1; echo "full rc=$?" >> $OUT/rc.txt ;;
  esac
done
