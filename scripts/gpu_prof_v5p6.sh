set -x
CMD="python tools/sw_probe.py"
export ONLY_SW=1 REPS=1
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_apply5" -s 20 -c 1 -o gpurun_out/prof_v5p6 -f $CMD > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
