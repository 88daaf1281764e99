# round-2 third session: where does the c5 solve and the c4 stage time go
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/pcg_breakdown.py 5 2>&1 | grep -v Warn
timeout 300 python tools/stage_one.py 2>&1 | grep -o "stage [0-9.]* ms.*" | cut -c1-400
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4_stage_launches.csv python tools/stage_one.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r4_stage_launches.csv | head -40
