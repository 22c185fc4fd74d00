for v in base fhw6 fhw7 fhw8; do
  echo "== $v"
  KIFMM_LIB=variants/$v.so timeout 300 python tools/near_time.py 2 30 2>&1 | tail -1 | cut -c1-90
  KIFMM_NEAR_BPS=0 KIFMM_LIB=variants/$v.so timeout 300 python tools/near_time.py 2 10 2>&1 | tail -1 | grep -o '"leaf_ms": [0-9.]*'
  KIFMM_LIB=variants/$v.so timeout 300 python tools/near_time.py 3 20 2>&1 | tail -1 | cut -c1-90
done
