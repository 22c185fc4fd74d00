KIFMM_CFG=4 KIFMM_ITERS=1 timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"m2l_oz_kernel|oz_slice|oz_level" -c 3 -o /tmp/oz4 python tools/profile_run.py > gpurun_out/ozncu.log 2>&1; echo rc=$?
ncu -i /tmp/oz4.ncu-rep --page raw --csv > gpurun_out/oz4_raw.csv 2>&1
ncu -i /tmp/oz4.ncu-rep --page source --csv --print-source sass -k regex:m2l_oz > gpurun_out/oz4_src.csv 2>&1
ls -la /tmp/oz4.ncu-rep; cp /tmp/oz4.ncu-rep gpurun_out/
