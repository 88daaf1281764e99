# DG div/grad at 3 CTAs per SM (80 registers) vs 2 (HEAD)
for i in 1 2; do DG_LIBRARY=$PWD/build_ab/libH1.so timeout 120 python tools/divgrad_time.py 2>&1 | grep -v Warn; timeout 120 python tools/divgrad_time.py 2>&1 | grep -v Warn; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "divergence" 2>&1 | tail -1
