# (1) v4 brick budget A/B for the variable-nu P = 7 solves of the VVP step (1x1x1 bricks at the 110 KB budget)
for kb in 110 160 227; do DG_LIBRARY=$PWD/build_ab/libDEV.so DG_SMEM_BUDGET_KB=$kb timeout 200 python tools/ab_p7nu.py 2>&1 | grep -v Warn | tail -1; done
timeout 200 python tools/ab_p7nu.py 2>&1 | grep -v Warn | tail -1
# (2) ncu of the Schwarz Poisson iteration's kernels and the velocity MODE-3 apply inside a config-4 stage
for k in "k_apply6<6" k_sw_block k_sw_pupd k_pcg_pupd_xt k_pcg_update_t "k_apply6<7, 0, 3"; do
  n=$(echo "$k" | tr -cd 'a-z0-9_'); 
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s 30 -c 1 -o gpurun_out/r5_$n python tools/stage_one.py > gpurun_out/r5_$n.log 2>&1; echo "$n rc=$?"
done
ls -la gpurun_out/*.ncu-rep
