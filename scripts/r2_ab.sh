for v in V26 V25; do DG_LIBRARY=$PWD/build_ab/lib$v.so timeout 300 python tools/slab_model.py 2>/dev/null; done
