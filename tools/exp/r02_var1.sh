# near-field variants: evaluate (queue mode) and serialized phases, configs 2 and 5
set -x
for v in base u8 il m10 m8 np2m8; do
  KIFMM_LIB=variants/$v.so timeout 300 python tools/near_time.py 2 30 2>&1 | tail -1
  KIFMM_NEAR_BPS=0 KIFMM_LIB=variants/$v.so timeout 300 python tools/near_time.py 2 10 2>&1 | tail -1
done
for v in base u8 il m10; do
  KIFMM_NEAR_BPS=0 KIFMM_LIB=variants/$v.so timeout 300 python tools/near_time.py 5 2 2>&1 | tail -1
done
