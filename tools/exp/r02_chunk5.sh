KIFMM_LIB=variants/base.so python tools/exp/cmp_lib.py 5 save /tmp/ref5.npz
KIFMM_LIB=variants/head.so python tools/exp/cmp_lib.py 5 check /tmp/ref5.npz 2>&1 | tail -1
KIFMM_LIB=variants/head.so timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-100
KIFMM_LIB=variants/base.so timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-100
