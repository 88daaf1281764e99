nvidia-smi --query-gpu=name,clocks.sm --format=csv
bash scripts/r3_ab.sh E0 E1 E2 E3 2>&1 | grep -v Warn
DG_LIBRARY=$PWD/build_ab/libE4.so timeout 300 python tools/v5_counters.py 2>&1 | tail -12
