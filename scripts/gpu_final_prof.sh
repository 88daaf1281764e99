# launch list of the default bench run (apply, PCG, stage) + one full ncu capture of the apply
CMD="python bench.py --steps 3 --warmup 3 --solves 1 --solve-warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_final.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD2="python bench.py --steps 3 --warmup 3 --solves 1 --solve-warmup 0 --no-cpu-baseline --no-stage"
ncu --set full --clock-control none --import-source on -k regex:"k_apply6|k_pcg_update_nox|k_pcg_pupd_x" -s 3 -c 3 -o gpurun_out/prof_final -f $CMD2 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
