timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gt1.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gt1.log
for c in 3 5; do python tools/near_time.py $c 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['cfg'], 'hw', round(d['ms_median'],3), d['leaf_ms'])"; KIFMM_FAR_HW=0 python tools/near_time.py $c 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['cfg'], 'f2', round(d['ms_median'],3), d['leaf_ms'])"; done
python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-90
