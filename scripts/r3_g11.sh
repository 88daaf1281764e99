timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py tests/test_gpu_schwarz.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
for v in N0 P0 P1 N0 P0 P1; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_apply.py 2>&1 | grep -v Warn; done
for v in N0 P0 P1; do echo $v; DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/pcg_breakdown.py 5 2>&1 | grep -v Warn | grep -E "maxit +(4|16|5000) "; done
for v in N0 P0 P1; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn | grep schwarz | cut -c1-120; done
