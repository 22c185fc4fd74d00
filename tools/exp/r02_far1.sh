timeout 600 python -m pytest tests/test_gpu.py -q -x -k "schedule_switches or far_pipe" -p no:cacheprovider 2>&1 | tail -3
for v in 1 0; do
  KIFMM_FAR_PIPE=$v timeout 300 python tools/near_time.py 2 30 2>&1 | tail -1 | cut -c1-400
done
for v in 1 0; do
  KIFMM_FAR_PIPE=$v timeout 300 python tools/near_time.py 3 20 2>&1 | tail -1 | cut -c1-400
  KIFMM_FAR_PIPE=$v timeout 300 python tools/near_time.py 5 2 2>&1 | tail -1 | cut -c1-400
done
