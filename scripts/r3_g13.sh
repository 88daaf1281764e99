timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_halo.py tests/test_gpu_schwarz.py -x -q 2>&1 | tail -3
for v in K1 S0 K1 S0; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn | grep -v "^P"; done
python tools/stage_one.py 2>&1 | grep -o "stage [0-9.]* ms"
