# ncu of the stage's remaining low-fraction kernels: convect (even-odd), DG divergence (padded), stabilisation apply
python tools/convect_time.py > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_convect3 -s 2 -c 1 -o gpurun_out/r4_convect python tools/convect_time.py > /dev/null 2>&1; echo cv $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dg_div2 -s 2 -c 1 -o gpurun_out/r4_div python tools/divgrad_time.py > /dev/null 2>&1; echo div $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stab_apply -s 2 -c 1 -o gpurun_out/r4_stab python tools/stab_time.py > /dev/null 2>&1; echo stab $?
python tools/stab_time.py 2>&1 | grep -v Warn
