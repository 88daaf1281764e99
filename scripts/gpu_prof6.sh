set -x
CMD="python bench.py --steps 3 --warmup 3 --solves 1 --solve-warmup 0 --no-cpu-baseline --no-stage"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_apply6" -s 3 -c 1 -o gpurun_out/prof_v6 -f $CMD > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
