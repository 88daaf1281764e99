# round-2 evidence: default bench line, launch list of the same command, one full ncu capture of the c5 apply
timeout 1500 python bench.py > gpurun_out/r3p_bench.json 2> gpurun_out/r3p_bench.err; echo bench rc=$?
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3p_launches.csv python bench.py --no-traffic --no-cpu-baseline > gpurun_out/r3p_ncu_launch.log 2>&1; echo launches rc=$?
python tools/one_apply.py 5 > gpurun_out/oa.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_apply6 -s 1 -c 1 -o gpurun_out/r3p_v6 python tools/one_apply.py 5 > gpurun_out/r3p_v6.log 2>&1; echo ncu rc=$?
