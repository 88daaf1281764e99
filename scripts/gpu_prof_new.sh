set -x
CMD="python tools/sw_probe.py"
export ONLY_SW=1 REPS=1
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sw_block|k_sw_pupd" -s 4 -c 2 -o gpurun_out/prof_sw2 -f $CMD > gpurun_out/ncu_full.log 2>&1
CMD2="python bench.py --steps 1 --warmup 3 --solves 1 --solve-warmup 0 --no-cpu-baseline"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_convect3" -s 1 -c 1 -o gpurun_out/prof_cv2 -f $CMD2 > gpurun_out/ncu_full2.log 2>&1
tail -2 gpurun_out/ncu_full.log gpurun_out/ncu_full2.log
