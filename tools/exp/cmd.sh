for v in base ws5 ws5u8 ws4u8; do KIFMM_LIB=variants/$v.so python tools/near_time.py 2 50 2>&1 | tail -1; done
KIFMM_NEAR_WS=0 KIFMM_LIB=variants/base.so python tools/near_time.py 2 50 2>&1 | tail -1
