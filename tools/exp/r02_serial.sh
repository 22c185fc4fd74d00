timeout 900 python -m pytest tests/test_gpu.py -q -x -k "queue_mode or schedule or smoke or parity_vs_oracle" -p no:cacheprovider 2>&1 | tail -1
for v in 0 1; do KIFMM_NEAR_SERIAL=$v timeout 600 python tools/near_time.py 4 5 2>&1 | tail -1 | cut -c1-100; done
for v in 0 1; do KIFMM_NEAR_SERIAL=$v timeout 600 python tools/near_time.py 2 30 2>&1 | tail -1 | cut -c1-100; done
