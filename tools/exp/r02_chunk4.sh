KIFMM_LIB=variants/base.so python tools/exp/cmp_lib.py 5 save /tmp/ref5.npz
for ch in 0 8; do KIFMM_FAR_CHUNK=$ch python tools/exp/cmp_lib.py 5 check /tmp/ref5.npz 2>&1 | tail -1; done
KIFMM_FAR_CHUNK=0 KIFMM_PLAN_TIMING=1 python tools/exp/cmp_lib.py 5 check /tmp/ref5.npz 2>&1 | tail -25
