timeout 900 python -m pytest tests/test_gpu.py -q -k "m2p_pass or parity_vs_oracle or two_cluster or sphere" -p no:cacheprovider 2>&1 | tail -2
for v in 1 0; do
  KIFMM_FAR_SPLIT=$v timeout 300 python tools/near_time.py 3 30 2>&1 | tail -1 | cut -c1-120
  KIFMM_FAR_SPLIT=$v timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-120
done
timeout 900 python -m pytest tests/test_gpu_configs.py -q -k "3 or 5" -p no:cacheprovider 2>&1 | tail -1
tail -2 gpurun_out/parity_r02.jsonl | cut -c1-250
