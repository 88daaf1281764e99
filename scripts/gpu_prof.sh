# ncu --set full capture of the apply (MODE 0 and PCG MODE 1) and the PCG update kernels (c5)
set -x
./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1; cat gpurun_out/fp64_peak.json
CMD="python bench.py --steps 3 --warmup 3 --solves 1 --solve-warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_apply|k_pcg_update" -s 5 -c 4 -o gpurun_out/prof_v4 -f $CMD > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
