timeout 900 python -m pytest tests/test_gpu.py -q -x -k "parity_vs_oracle or queue or schedule or two_cluster" > gpurun_out/t9.log 2>&1; echo t rc=$?; tail -2 gpurun_out/t9.log
rm -f gpurun_out/parity_r02.jsonl
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "3 or 5" > gpurun_out/t9c.log 2>&1; echo tc rc=$?; tail -2 gpurun_out/t9c.log
for o in 1 0; do KIFMM_P2L_OVERLAP=$o python tools/near_time.py 3 20 2>&1 | tail -1; KIFMM_P2L_OVERLAP=$o python tools/near_time.py 5 3 2>&1 | tail -1; done
for f in 0 1; do KIFMM_NEAR_BPS=2 python tools/near_time.py 5 3 2>&1 | tail -1; done
