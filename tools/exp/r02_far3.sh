KIFMM_NEAR_BPS=0 KIFMM_CFG=3 KIFMM_ITERS=1 timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"far_hw" -c 1 -o /tmp/f3 python tools/profile_run.py > gpurun_out/f3.log 2>&1; echo rc=$?
ncu -i /tmp/f3.ncu-rep --page raw --csv > gpurun_out/f3_raw.csv 2>&1
ncu -i /tmp/f3.ncu-rep --page source --csv --print-source sass > gpurun_out/f3_src.csv 2>&1
