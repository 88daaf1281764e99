# round-2 final validation of HEAD: smoke, every GPU test, default bench line, reference arm,
# launch list of the default bench, one full ncu capture of the c5 apply
set -x
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/r5h_smoke.log 2>&1; tail -2 gpurun_out/r5h_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r5h_gpu_tests.log 2>&1; tail -3 gpurun_out/r5h_gpu_tests.log
timeout 1500 python bench.py > gpurun_out/r5h_bench.json 2> gpurun_out/r5h_bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r5h_ref.json 2> gpurun_out/r5h_ref.err; echo ref rc=$?
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5h_launches.csv python bench.py --no-traffic --no-cpu-baseline > gpurun_out/r5h_ncu_launch.log 2>&1; echo launches rc=$?
python tools/one_apply.py 5 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_apply6 -s 1 -c 1 -o gpurun_out/r5h_v6 python tools/one_apply.py 5 > gpurun_out/r5h_v6.log 2>&1; echo ncu rc=$?
