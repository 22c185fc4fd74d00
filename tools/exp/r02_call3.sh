set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cli.py tests/test_gpu_acceptance.py -m gpu -q -rf -p no:cacheprovider > gpurun_out/t3.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/t3.log
for c in 2 3 5; do KIFMM_CFG=$c KIFMM_ITERS=3 timeout 600 python tools/profile_run.py > gpurun_out/prof$c.log 2>&1; echo prof$c rc=$?; done
for c in 2 5; do
KIFMM_NEAR_BPS=0 KIFMM_CFG=$c KIFMM_ITERS=1 timeout 1200 ncu -f --set full --clock-control none --import-source on \
  -k regex:"leaf_eval|far_hw|far_f2|check_f2" -c 4 -o /tmp/r02n_cfg$c python tools/profile_run.py > gpurun_out/ncun$c.log 2>&1
echo ncu$c rc=$?
ncu -i /tmp/r02n_cfg$c.ncu-rep --page raw --csv > gpurun_out/r02n_cfg${c}_raw.csv 2>&1
ncu -i /tmp/r02n_cfg$c.ncu-rep --page source --csv --print-source sass > gpurun_out/r02n_cfg${c}_src.csv 2>&1
ls -la /tmp/r02n_cfg$c.ncu-rep
done
cp /tmp/r02n_cfg2.ncu-rep gpurun_out/
du -sh gpurun_out
