timeout 900 python -m pytest tests/test_gpu.py -q -k "fp64 or tiny or small_trees or coincident or single_leaf or run_api" -p no:cacheprovider 2>&1 | tail -1
for v in 1 0; do KIFMM_NEAR_PAIR64=$v timeout 600 python tools/near_time.py 4 5 2>&1 | tail -1 | cut -c1-320; done
timeout 900 python -m pytest tests/test_gpu_configs.py -q -k "4" -p no:cacheprovider 2>&1 | tail -1
