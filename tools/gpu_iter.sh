# One build -> measure iteration on the GPU box: parity subset, config-2 / config-4 bench lines,
# one --set full capture of the kernels matching $KREG. Outputs under gpurun_out/$T/.
T=${T:-r02x}
KREG=${KREG:-raster_bwd_kernel}
mkdir -p gpurun_out/$T
python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py tests/test_gpu_decoder_oracle.py tests/test_gpu_sharded.py tests/test_gpu_decoder_tc.py -x -q > gpurun_out/$T/tests.log 2>&1; echo tests=$?
python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/$T/c2.json 2>gpurun_out/$T/c2.err; echo c2=$?
python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c4.json 2>gpurun_out/$T/c4.err; echo c4=$?
ncu --kernel-name regex:"$KREG" --launch-skip 20 -c ${KCOUNT:-1} --set full --import-source on --clock-control none -o gpurun_out/$T/prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-phases 0 > gpurun_out/$T/ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/$T/tests.log
