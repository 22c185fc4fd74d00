timeout 300 python -m pytest tests/test_gpu.py -x -q -k "queue_mode or parity_vs_oracle or config2_full or evaluate_many" > gpurun_out/gt1.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gt1.log
for i in 1 2 3; do python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-80; KIFMM_NEAR_WS=0 python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-80; done
