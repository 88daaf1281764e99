timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py -x -q -k "apply or diag or v6 or pcg" 2>&1 | tail -3
bash scripts/r3_ab.sh G3 H0 H1 H2 H5 2>&1 | grep -v Warn
DG_LIBRARY=$PWD/build_ab/libH4.so timeout 300 python tools/v5_counters.py 2>&1 | tail -11
