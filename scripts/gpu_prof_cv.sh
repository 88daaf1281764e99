set -x
CMD="python bench.py --steps 1 --warmup 3 --solves 1 --solve-warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_convect3" -s 1 -c 1 -o gpurun_out/prof_cv -f $CMD > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
