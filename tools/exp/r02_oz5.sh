rm -f gpurun_out/ozaki_r02.jsonl
timeout 900 python -m pytest tests/test_gpu.py -q -k "ozaki or int8 or (parity_vs_oracle and fp64) or fp64" -p no:cacheprovider 2>&1 | tail -2
cat gpurun_out/ozaki_r02.jsonl
timeout 600 python tools/near_time.py 4 5 2>&1 | tail -1 | cut -c1-400
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "4" -p no:cacheprovider 2>&1 | tail -1
tail -1 gpurun_out/parity_r02.jsonl
