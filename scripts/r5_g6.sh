# P = 7 v6 apply: SE = 514 / rows 4 SE apart (conflict-free x, y, z passes in the bank model) and 16-byte x-pass stores for
# constant nu: A/B vs the previous commit (libH3), parity
for i in 1 2; do DG_LIBRARY=$PWD/build_ab/libH3.so timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn | tail -1; timeout 300 python tools/ab_c4.py 2>&1 | grep -v Warn | tail -1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c4 or stage or c3 or apply_every" 2>&1 | tail -2
timeout 300 python tools/stage_one.py 2>&1 | grep -o "stage [0-9.]* ms"
