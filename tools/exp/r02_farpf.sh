for c in 2 3; do
  KIFMM_LIB=variants/base.so python tools/exp/cmp_lib.py $c save /tmp/ref$c.npz
  python tools/exp/cmp_lib.py $c check /tmp/ref$c.npz 2>&1 | tail -1
done
for c in 2 3; do
  KIFMM_LIB=variants/base.so timeout 300 python tools/near_time.py $c 30 2>&1 | tail -1 | cut -c1-90
  timeout 300 python tools/near_time.py $c 30 2>&1 | tail -1 | cut -c1-90
done
KIFMM_LIB=variants/base.so timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-90
timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-90
KIFMM_NEAR_BPS=0 KIFMM_LIB=variants/base.so timeout 300 python tools/near_time.py 3 10 2>&1 | tail -1 | grep -o '"leaf_ms": [0-9.]*'
KIFMM_NEAR_BPS=0 timeout 300 python tools/near_time.py 3 10 2>&1 | tail -1 | grep -o '"leaf_ms": [0-9.]*'
