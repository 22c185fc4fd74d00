timeout 900 python -m pytest tests/test_gpu.py -q -k "ozaki or int8" -p no:cacheprovider -s 2>&1 | grep -E "^ozaki|passed|failed" | head -30
