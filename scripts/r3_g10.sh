timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py -x -q -k "apply or v6 or pcg or halo" 2>&1 | tail -3
for v in N0 O0 N0 O0; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_apply.py 2>&1 | grep -v Warn; done
DG_LIBRARY=$PWD/build_ab/libO4.so timeout 300 python tools/v5_counters.py 2>&1 | tail -11
