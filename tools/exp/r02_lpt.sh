for c in 2 3; do KIFMM_LIB=variants/head.so python tools/exp/cmp_lib.py $c save /tmp/ref$c.npz; python tools/exp/cmp_lib.py $c check /tmp/ref$c.npz 2>&1 | tail -1; done
for v in 1 0 1 0; do KIFMM_NEAR_LPT=$v timeout 300 python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-80; done
for v in 1 0; do KIFMM_NEAR_LPT=$v timeout 300 python tools/near_time.py 3 30 2>&1 | tail -1 | cut -c1-80; KIFMM_NEAR_LPT=$v KIFMM_NEAR_BPS=0 timeout 300 python tools/near_time.py 2 10 2>&1 | tail -1 | grep -o '"leaf_ms": [0-9.]*'; done
