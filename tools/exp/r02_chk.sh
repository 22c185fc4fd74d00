for c in 2 3 5; do KIFMM_LIB=variants/head.so python tools/exp/cmp_lib.py $c save /tmp/ref$c.npz; python tools/exp/cmp_lib.py $c check /tmp/ref$c.npz 2>&1 | tail -1; done
for v in 1 0; do for c in 2 3; do KIFMM_CHECK_HW=$v timeout 300 python tools/near_time.py $c 30 2>&1 | tail -1 | cut -c1-140; done; KIFMM_CHECK_HW=$v timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-140; done
for v in 1 0; do KIFMM_CHECK_HW=$v KIFMM_CFG=2 KIFMM_ITERS=1 timeout 300 ncu --metrics gpu__time_duration.sum -k regex:check python tools/profile_run.py 2>&1 | grep -E "check|duration" | head -4; done
