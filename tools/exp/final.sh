# Round-end evidence run on the GPU box: gpu tests, smoke, bench (+ reference arm), launch list, ncu --set full capture.
# usage: gpurun -- bash tools/exp/final.sh   (outputs under gpurun_out/)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; cat gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log > gpurun_out/bench_line.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
KIFMM_NEAR_BPS=0 KIFMM_ITERS=1 timeout 1200 ncu --set full --clock-control none --import-source on -c 24 -o gpurun_out/full python tools/profile_run.py > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
