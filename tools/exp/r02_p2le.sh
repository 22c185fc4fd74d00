for c in 3 5; do KIFMM_LIB=variants/head.so python tools/exp/cmp_lib.py $c save /tmp/ref$c.npz; python tools/exp/cmp_lib.py $c check /tmp/ref$c.npz 2>&1 | tail -1; done
for v in 1 0; do KIFMM_P2L_EARLY=$v timeout 300 python tools/near_time.py 3 30 2>&1 | tail -1 | cut -c1-80; KIFMM_P2L_EARLY=$v timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-80; done
