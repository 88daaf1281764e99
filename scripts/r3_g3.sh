timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "apply or diag or c5 or helmholtz" 2>&1 | tail -3
bash scripts/r3_ab.sh E0 F0 F1 2>&1 | grep -v Warn
DG_LIBRARY=$PWD/build_ab/libF4.so timeout 300 python tools/v5_counters.py 2>&1 | tail -11
