timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py -x -q -k "diag or pcg or helmholtz" 2>&1 | tail -3
python tools/diag_time.py 5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_diag_cf3 -s 3 -c 1 -o gpurun_out/r3_diag python tools/diag_time.py 5 > gpurun_out/r3_diag.log 2>&1; echo ncu rc=$?
