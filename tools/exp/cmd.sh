timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gputests.log
for i in 1 2; do python tools/near_time.py 2 50 2>&1 | tail -1; KIFMM_NEAR_WS=1 python tools/near_time.py 2 50 2>&1 | tail -1; done
KIFMM_NEAR_BPS=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:leaf_eval_f2 -c 1 -o gpurun_out/near2 python tools/profile_run.py > gpurun_out/ncu_near.log 2>&1; echo ncu rc=$?
