# even-odd convection: parity and time
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "convect" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k "convect" 2>&1 | tail -2
timeout 300 python tools/convect_time.py 2>&1 | grep -v Warn
timeout 300 python tools/convect_time.py 2>&1 | grep -v Warn
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "apply_diag_small" 2>&1 | tail -2
