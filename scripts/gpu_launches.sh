# per-launch device times of one bench run (cold-cache, serialised: compare shares)
CMD="python bench.py --steps 3 --warmup 3 --solves 1 --solve-warmup 0 --no-cpu-baseline --no-stage"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
