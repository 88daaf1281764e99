timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py tests/test_gpu_schwarz.py -x -q 2>&1 | tail -3
for v in L0 N0 N1 N2 L0 N0; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_apply.py 2>&1 | grep -v Warn; done
for v in L0 N0 N1 N2; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn | grep -v "^ \|Trace\|Error" | cut -c1-110; done
DG_LIBRARY=$PWD/build_ab/libN4.so timeout 300 python tools/v5_counters.py 2>&1 | tail -11
