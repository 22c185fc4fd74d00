timeout 600 python -m pytest tests/test_gpu.py -x -q -k "dmma" > gpurun_out/gt1.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gt1.log
python tools/near_time.py 4 5 2>&1 | tail -1
KIFMM_CFG=4 KIFMM_ITERS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_dmma -s 6 -c 1 -o gpurun_out/dmma2 python tools/profile_run.py > gpurun_out/ncu_dmma.log 2>&1; echo ncu rc=$?
