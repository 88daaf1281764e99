# ncu of the config-4 stage applies, summarised on the box (the reports with sources exceed the copy-back limit)
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_apply6<\(int\)6' -s 30 -c 1 -o /tmp/r5_apply6_p6 python tools/stage_one.py > gpurun_out/r5_apply6_p6.log 2>&1; echo "p6 rc=$?"
python tools/ncu_summary.py /tmp/r5_apply6_p6.ncu-rep "v6::k_apply6<6,0,2> (P = 6 pressure apply with the dot epilogue) inside a config-4 stage, 32^3 elements" 179830784 > gpurun_out/r02c_apply6_p6_ncu.json
ncu -i /tmp/r5_apply6_p6.ncu-rep --page source --csv --print-source cuda,sass > /tmp/p6src.csv 2>/dev/null; gzip -c /tmp/p6src.csv > gpurun_out/r5_apply6_p6_src.csv.gz
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_apply6<\(int\)7, \(bool\)0, \(int\)3' -s 10 -c 1 -o /tmp/r5_apply6_p7 python tools/stage_one.py > gpurun_out/r5_apply6_p7.log 2>&1; echo "p7 rc=$?"
python tools/ncu_summary.py /tmp/r5_apply6_p7.ncu-rep "v6::k_apply6<7,0,3> (P = 7 velocity Helmholtz apply with the dot epilogue) inside a config-4 stage, 32^3 elements" 268435456 > gpurun_out/r02c_apply6_p7_ncu.json
ls -la gpurun_out
