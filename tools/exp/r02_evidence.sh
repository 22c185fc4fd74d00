# Evidence run on the GPU box (outputs under gpurun_out/, kept well under gpurun's 64 MiB pull limit:
# ncu reports go to /tmp and only CSV exports + the small per-config reports come back).
# usage: gpurun -- bash tools/exp/r02_evidence.sh [tests] [bench] [ncu]
set -x
mkdir -p gpurun_out
want() { [ $# -eq 0 ] || [[ " $ARGS " == *" $1 "* ]]; }
ARGS="$*"
if [[ -z "$ARGS" || " $ARGS " == *" tests "* ]]; then
  timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests rc=$?
  tail -15 gpurun_out/gputests.log
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; cat gpurun_out/smoke.log
fi
if [[ -z "$ARGS" || " $ARGS " == *" bench "* ]]; then
  python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log > gpurun_out/bench_line.json
  cat gpurun_out/bench_line.json
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
fi
if [[ -z "$ARGS" || " $ARGS " == *" ncu "* ]]; then
  for c in ${NCU_CFGS:-2 3 5}; do
    KIFMM_NEAR_BPS=0 KIFMM_CFG=$c KIFMM_ITERS=1 timeout 1200 ncu -f --set full --clock-control none --import-source on \
      -k regex:"leaf_eval|far_hw|far_f2|check_f2|m2l_tc_kernel<160, 1|near_ws|gather_dmma" -c ${NCU_COUNT:-8} -o /tmp/r02_cfg$c \
      python tools/profile_run.py > gpurun_out/ncu$c.log 2>&1
    echo cfg$c rc=$?
    ncu -i /tmp/r02_cfg$c.ncu-rep --page raw --csv > gpurun_out/r02_cfg${c}_raw.csv 2>&1
    ncu -i /tmp/r02_cfg$c.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_cfg${c}_src.csv 2>&1
    ls -la /tmp/r02_cfg$c.ncu-rep
    sz=$(stat -c %s /tmp/r02_cfg$c.ncu-rep)
    [ "$sz" -lt 20000000 ] && cp /tmp/r02_cfg$c.ncu-rep gpurun_out/
  done
fi
du -sh gpurun_out
