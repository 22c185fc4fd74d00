timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gt1.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gt1.log
for i in 1 2; do python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-100; KIFMM_LIB=variants/base.so python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-100; done
for c in 3 5; do python tools/near_time.py $c 10 2>&1 | tail -1 | cut -c1-70; done
