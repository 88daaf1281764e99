# P = 6 v6 apply: permuted line order in the x and y passes (bank conflicts of the dense row-TMA slots): A/B vs HEAD (libH2), parity
for i in 1 2; do DG_LIBRARY=$PWD/build_ab/libH2.so timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn | tail -1; timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn | tail -1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schwarz.py tests/test_gpu_halo.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "schwarz or stage or c3" 2>&1 | tail -2
timeout 300 python tools/stage_one.py 2>&1 | grep -o "stage [0-9.]* ms"
