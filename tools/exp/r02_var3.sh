for e in "KIFMM_X=0" "KIFMM_NEAR_SKIP=1" "KIFMM_NEAR_BPS=1" "KIFMM_NEAR_BPS=0"; do
  echo "== $e"
  env $e KIFMM_LIB=variants/tl.so KIFMM_TIMELINE=1 KIFMM_NEAR_DEBUG=1 timeout 300 python tools/timeline.py 2 2>&1 | tail -7
done
