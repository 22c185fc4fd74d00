KIFMM_NEAR_BPS=0 KIFMM_CFG=3 KIFMM_ITERS=1 timeout 1200 ncu -f --set full --clock-control none -k regex:"leaf_eval|far_hw|far_f2|check_f2|m2l_tc_kernel<1" -c 5 -o /tmp/r02n_cfg3 python tools/profile_run.py > gpurun_out/ncun3.log 2>&1; echo rc=$?
ncu -i /tmp/r02n_cfg3.ncu-rep --page raw --csv > gpurun_out/r02n_cfg3_raw.csv 2>&1
KIFMM_CFG=2 KIFMM_ITERS=1 timeout 1200 ncu -f --set full --clock-control none -k regex:"m2l_tc_kernel<1|near_ws" -c 2 -o /tmp/r02m_cfg2 python tools/profile_run.py > gpurun_out/ncum2.log 2>&1; echo rc=$?
ncu -i /tmp/r02m_cfg2.ncu-rep --page raw --csv > gpurun_out/r02m_cfg2_raw.csv 2>&1
ls -la /tmp/*.ncu-rep
