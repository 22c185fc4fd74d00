for e in "KIFMM_X=0" "KIFMM_NEAR_WARP=1"; do
  echo "== $e"
  env $e timeout 300 python tools/near_time.py 2 30 2>&1 | tail -1 | cut -c1-90
  env $e KIFMM_NEAR_BPS=0 timeout 300 python tools/near_time.py 2 10 2>&1 | tail -1 | grep -o '"leaf_ms": [0-9.]*'
  env $e timeout 300 python tools/near_time.py 3 20 2>&1 | tail -1 | cut -c1-90
  env $e KIFMM_NEAR_BPS=0 timeout 300 python tools/near_time.py 3 10 2>&1 | tail -1 | grep -o '"leaf_ms": [0-9.]*'
done
