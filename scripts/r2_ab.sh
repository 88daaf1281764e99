for v in V22 V27 V22 V27; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/ab_apply.py; done
