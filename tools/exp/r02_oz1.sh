timeout 900 python -m pytest tests/test_gpu.py -q -x -k "ozaki or int8 or (parity_vs_oracle and fp64)" -p no:cacheprovider -s 2>&1 | grep -E "ozaki|passed|failed|Error|error" | head -30
timeout 600 python tools/near_time.py 4 3 2>&1 | tail -1 | cut -c1-400
KIFMM_M2L_BACKEND=1 timeout 600 python tools/near_time.py 4 3 2>&1 | tail -1 | cut -c1-400
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "4" -p no:cacheprovider 2>&1 | tail -3
tail -2 gpurun_out/parity_r02.jsonl
