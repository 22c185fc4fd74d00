for v in 1 0; do echo "== split $v"; KIFMM_FAR_SPLIT=$v KIFMM_LIB=variants/tl.so KIFMM_TIMELINE=1 KIFMM_NEAR_DEBUG=1 timeout 300 python tools/timeline.py 3 2>&1 | tail -8; done
