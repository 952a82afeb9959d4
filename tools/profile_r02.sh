#!/bin/bash
# Round-2 profile captures on the GPU box (run each after the plain command exits 0; never a
# multi-rank command). Outputs under gpurun_out/r02p/; summaries go to profiles/ by hand.
set -x
OUT=gpurun_out/r02p
mkdir -p $OUT
DEC="sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.sum,sm__ops_path_tensor_op_hmma_src_fp16_dst_fp32.sum,sm__inst_executed_pipe_tc.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/plain_c2.json 2>&1 || exit 1
# 1) launch list of one config-2 step (cold, serialised per-launch times)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-phases 0 > $OUT/ncu_launch.log 2>&1
# 2) decoder tensor-pipe metrics, config 2 (fused DEC1/DEC2) and config 4 (staged DL1-DL5)
ncu --kernel-name regex:"dec1_kernel|dec2_kernel|dec_reduce|dl_" --metrics $DEC --clock-control none -c 40 --csv \
    --log-file $OUT/decoder_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-phases 0 > $OUT/ncu_dec2.log 2>&1
python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $OUT/plain_c4.json 2>&1
ncu --kernel-name regex:"dl_" --metrics $DEC --clock-control none -c 40 --csv \
    --log-file $OUT/decoder_c4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --profile-phases 0 > $OUT/ncu_dec4.log 2>&1
# 3) full set of the raster kernels (one launch each)
ncu --kernel-name regex:"raster_bwd_kernel|raster_fwd_mma_kernel" --launch-skip 30 -c 2 --set full --import-source on \
    --clock-control none -o $OUT/raster_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-phases 0 > $OUT/ncu_raster.log 2>&1
ls -la $OUT
