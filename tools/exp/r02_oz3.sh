rm -f gpurun_out/ozaki_r02.jsonl
timeout 900 python -m pytest tests/test_gpu.py -q -k "ozaki" -p no:cacheprovider 2>&1 | tail -1
KIFMM_LIB=variants/oz8.so timeout 900 python -m pytest tests/test_gpu.py -q -k "ozaki" -p no:cacheprovider 2>&1 | tail -1
cat gpurun_out/ozaki_r02.jsonl
KIFMM_LIB=variants/oz8.so timeout 600 python tools/near_time.py 4 3 2>&1 | tail -1 | cut -c1-300
