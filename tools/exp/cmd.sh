KIFMM_LIB=variants/rcp.so timeout 300 python -m pytest tests/test_gpu.py -x -q -k "parity_vs_oracle or config2_full or queue_mode" 2>&1 | tail -2
for v in base rcp base rcp; do KIFMM_LIB=variants/$v.so python tools/near_time.py 2 40 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['lib'], round(d['ms_median'],4), d['leaf_ms'])"; done
