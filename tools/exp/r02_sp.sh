KIFMM_LIB=variants/base.so python tools/exp/cmp_lib.py 2 save /tmp/ref2.npz
for v in base sp spm8 spm7; do
  echo "== $v"
  KIFMM_LIB=variants/$v.so python tools/exp/cmp_lib.py 2 check /tmp/ref2.npz 2>&1 | tail -1
  KIFMM_NEAR_BPS=0 KIFMM_LIB=variants/$v.so timeout 300 python tools/near_time.py 2 10 2>&1 | tail -1 | grep -o '"leaf_ms": [0-9.]*'
  KIFMM_LIB=variants/$v.so timeout 300 python tools/near_time.py 2 30 2>&1 | tail -1 | cut -c1-90
  KIFMM_NEAR_BPS=0 KIFMM_LIB=variants/$v.so timeout 300 python tools/near_time.py 5 2 2>&1 | tail -1 | grep -o '"leaf_ms": [0-9.]*'
done
