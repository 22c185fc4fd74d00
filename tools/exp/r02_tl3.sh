KIFMM_LIB=variants/tl.so KIFMM_TIMELINE=1 KIFMM_NEAR_DEBUG=1 timeout 600 python tools/timeline.py 3 2>&1 | tail -8
KIFMM_LIB=variants/tl.so KIFMM_TIMELINE=1 KIFMM_NEAR_DEBUG=1 timeout 600 python tools/timeline.py 2 2>&1 | tail -8
