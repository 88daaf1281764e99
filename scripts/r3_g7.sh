timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schwarz.py tests/test_gpu_halo.py -x -q -k "small or schwarz or poisson or c3 or c4" 2>&1 | tail -3
for v in K1 K0 K1 K0; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn; done
