KIFMM_CFG=4 KIFMM_ITERS=1 timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"leaf_eval|far_kernel|check_kernel" -c 4 -o /tmp/c4p python tools/profile_run.py > gpurun_out/ncu4p.log 2>&1; echo rc=$?
ncu -i /tmp/c4p.ncu-rep --page raw --csv > gpurun_out/c4p_raw.csv 2>&1
ncu -i /tmp/c4p.ncu-rep --page source --csv --print-source sass -k regex:leaf_eval > gpurun_out/c4p_src.csv 2>&1
