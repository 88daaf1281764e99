# A/B: v6 P = 6 brick rows (4 / 2) and register cap (80 / 96)
for v in K0 R96 B2 B2R; do echo "== $v"; DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 120 python tools/ab_check67.py 2>&1 | grep -v Warn; done
for v in K0 R96 B2 B2R K0 R96 B2 B2R; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn | grep -v "^P"; done
