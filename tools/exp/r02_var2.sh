set -x
KIFMM_LIB=variants/tl.so KIFMM_TIMELINE=1 KIFMM_NEAR_DEBUG=1 timeout 300 python tools/timeline.py 2 2>&1 | tail -12
KIFMM_LIB=variants/tl.so KIFMM_TIMELINE=1 KIFMM_NEAR_DEBUG=1 timeout 300 python tools/timeline.py 3 2>&1 | tail -12
for e in "KIFMM_NEAR_SKIP=1" "KIFMM_NEAR_BPS=1" "KIFMM_NEAR_BPS=3" "KIFMM_NEAR_WS=0" "KIFMM_NEAR_PAUSE=1" "KIFMM_NEAR_PAUSE=2"; do
  env $e KIFMM_LIB=variants/base.so timeout 300 python tools/near_time.py 2 30 2>&1 | tail -1 | cut -c1-120
done
