timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py -x -q -k "diag or pcg or helmholtz" 2>&1 | tail -3
python tools/diag_time.py 5; python tools/diag_time.py 5
