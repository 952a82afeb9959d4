T=${T:-r02w}
mkdir -p gpurun_out/$T
python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py tests/test_gpu_decoder_oracle.py tests/test_gpu_sharded.py -x -q > gpurun_out/$T/tests.log 2>&1; echo tests=$?
python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/$T/c2.json 2>gpurun_out/$T/c2.err; echo c2=$?
python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c4.json 2>gpurun_out/$T/c4.err; echo c4=$?
ncu --kernel-name regex:raster_bwd_kernel --launch-skip 20 -c 1 --set full --import-source on --clock-control none -o gpurun_out/$T/bwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-phases 0 > gpurun_out/$T/ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/$T/tests.log
