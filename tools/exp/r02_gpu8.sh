for v in default il1 default il1; do
  if [ $v = default ]; then L=""; else L="variants/$v.so"; fi
  echo "== $v"; KIFMM_LIB=$L KIFMM_NEAR_BPS=0 python tools/near_time.py 2 30 2>&1 | tail -1
  KIFMM_LIB=$L python tools/near_time.py 2 30 2>&1 | tail -1
done
for v in default il1; do
  if [ $v = default ]; then L=""; else L="variants/$v.so"; fi
  KIFMM_LIB=$L python tools/near_time.py 3 20 2>&1 | tail -1; KIFMM_LIB=$L python tools/near_time.py 5 3 2>&1 | tail -1
done
