# Round-2 evidence run on the GPU box (outputs under gpurun_out/, small files only).
set -x
mkdir -p gpurun_out
rm -f gpurun_out/parity_r02.jsonl gpurun_out/ozaki_r02.jsonl gpurun_out/acceptance_r02.jsonl
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/f_gputests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/f_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke rc=$?; cat gpurun_out/f_smoke.log
python bench.py > gpurun_out/f_bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/f_bench.log > gpurun_out/f_bench_line.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_bench_ref.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/f_bench_ref.log > gpurun_out/f_bench_ref_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f_ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 python tools/configs.py > gpurun_out/f_configs.jsonl 2> gpurun_out/f_configs.err; echo configs rc=$?
du -sh gpurun_out
