timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "apply_diag_small or v6 or configs" 2>&1 | tail -2
for v in N0 Q1 N0 Q1; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_apply.py 2>&1 | grep -v Warn; done
for v in N0 Q1; do echo $v; DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/pcg_breakdown.py 5 2>&1 | grep -v Warn | grep -E "maxit +(4|16|5000) "; done
