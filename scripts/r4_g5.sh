# padded DG div/grad: parity and time (baseline lib built from HEAD for the A/B)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "divergence or imex_stage_small or rk_step_small" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "imex_stage" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_stab.py tests/test_gpu_halo.py -q -x 2>&1 | tail -2
for i in 1 2; do DG_LIBRARY=$PWD/build_ab/libH0.so timeout 120 python tools/divgrad_time.py 2>&1 | grep -v Warn; timeout 120 python tools/divgrad_time.py 2>&1 | grep -v Warn; done
timeout 300 python tools/stage_one.py 2>&1 | grep -o "stage [0-9.]* ms"
