set -x
for c in 2 3 5; do
KIFMM_CFG=$c KIFMM_ITERS=1 timeout 600 python tools/profile_run.py > gpurun_out/p$c.log 2>&1 && \
KIFMM_CFG=$c KIFMM_ITERS=1 timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"leaf_eval|far_hw|far_f2|check_f2|m2l_tc_kernel|near_ws" -c 12 -o /tmp/r02_cfg$c python tools/profile_run.py > gpurun_out/ncu$c.log 2>&1
echo cfg$c rc=$?
ncu -i /tmp/r02_cfg$c.ncu-rep --page raw --csv > gpurun_out/r02_cfg${c}_raw.csv 2>&1
for k in leaf_eval far_hw far_f2 check_f2 near_ws; do
  ncu -i /tmp/r02_cfg$c.ncu-rep --page source --csv -k regex:$k --launch-count 1 > gpurun_out/r02_cfg${c}_src_$k.csv 2>/dev/null
done
ls -la /tmp/r02_cfg$c.ncu-rep
done
cp /tmp/r02_cfg2.ncu-rep gpurun_out/ 2>/dev/null
du -sh gpurun_out; ls -la gpurun_out
