for b in 1 2; do echo "ws bps=$b"; KIFMM_NEAR_BPS=$b python tools/near_time.py 2 60 2>&1 | tail -1 | cut -c1-90; done
for b in 2 3 4; do echo "old bps=$b"; KIFMM_NEAR_WS=0 KIFMM_NEAR_BPS=$b python tools/near_time.py 2 60 2>&1 | tail -1 | cut -c1-90; done
echo "ws bps=2 pause2"; KIFMM_NEAR_PAUSE=2 python tools/near_time.py 2 60 2>&1 | tail -1 | cut -c1-90
