timeout 900 python tools/tg_final.py 8 2>&1 | grep -v Warn
timeout 300 python tools/stage_one.py 2>&1 | grep -o "stage [0-9.]* ms"
