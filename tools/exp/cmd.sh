timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gt1.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gt1.log
for i in 1 2; do python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-100; KIFMM_FAR_HW=0 python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-100; done
KIFMM_NEAR_BPS=0 KIFMM_ITERS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:far_hw -c 1 -o gpurun_out/farhw python tools/profile_run.py > gpurun_out/ncu_far.log 2>&1; echo ncu rc=$?
