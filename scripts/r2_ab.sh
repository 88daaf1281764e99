for v in V13 V11 V12 V13 V11 V12; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_apply.py; done
