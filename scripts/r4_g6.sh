# fused cluster coarse solve: parity (Schwarz tests) and time
timeout 900 python -m pytest tests/test_gpu_schwarz.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "schwarz or imex_stage or c3_poisson" 2>&1 | tail -2
for i in 1 2; do DG_LIBRARY=$PWD/build_ab/libH0.so timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn | grep -v "^P"; timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn | grep -v "^P"; done
timeout 300 python tools/stage_one.py 2>&1 | grep -o "stage [0-9.]* ms"
