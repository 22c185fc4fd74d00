for e in "KIFMM_NEAR_FORK=m2l" "KIFMM_NEAR_FORK=m2l KIFMM_NEAR_BPS=1"; do
  echo "== $e"
  env $e KIFMM_LIB=variants/tl.so KIFMM_TIMELINE=1 KIFMM_NEAR_DEBUG=1 timeout 300 python tools/timeline.py 2 2>&1 | tail -7
  env $e KIFMM_LIB=variants/base.so timeout 300 python tools/near_time.py 2 30 2>&1 | tail -1 | cut -c1-100
done
KIFMM_LIB=variants/base.so timeout 300 python tools/near_time.py 2 30 2>&1 | tail -1 | cut -c1-100
