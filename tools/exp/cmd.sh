timeout 300 python -m pytest tests/test_gpu.py -x -q -k "parity_vs_oracle" > gpurun_out/gt1.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gt1.log
KIFMM_M2M=parent timeout 300 python -m pytest tests/test_gpu.py -x -q -k "parity_vs_oracle or config2_full" > gpurun_out/gt2.log 2>&1; echo parent-tests rc=$?; tail -2 gpurun_out/gt2.log
for i in 1 2; do python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-100; KIFMM_M2M=parent python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-100; done
