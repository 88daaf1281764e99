timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py tests/test_gpu_schwarz.py -x -q 2>&1 | tail -3
for v in J0 L0 J0 L0; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_apply.py 2>&1 | grep -v Warn; done
for ns in 2 4 8 16; do echo nseg $ns; DG_V6_NSEG=$ns DG_LIBRARY=$PWD/build_ab/libL1.so timeout 300 python tools/ab_apply.py 2>&1 | grep -v Warn; done
for v in K1 L0; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn; done
for ns in 1 2 4 8; do echo nseg $ns; DG_V6_NSEG=$ns DG_LIBRARY=$PWD/build_ab/libL1.so timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn; done
