timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "apply_diag_small or configs_sampled" 2>&1 | tail -3
python tools/diag_time.py 5; DG_LIBRARY=$PWD/build_ab/libE0.so python tools/diag_time.py 5
python tools/diag_time.py 5
python tools/one_apply.py 5 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_apply6 -s 1 -c 1 -o gpurun_out/r3_v6 python tools/one_apply.py 5 > gpurun_out/r3_v6.log 2>&1; echo ncu rc=$?
