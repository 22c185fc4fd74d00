set -x
for c in 2 5; do
KIFMM_NEAR_BPS=0 KIFMM_CFG=$c KIFMM_ITERS=1 timeout 600 python tools/profile_run.py > gpurun_out/p$c.log 2>&1 && \
KIFMM_NEAR_BPS=0 KIFMM_CFG=$c KIFMM_ITERS=1 timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"leaf_eval|far_hw|far_f2" -c 2 -o /tmp/r02p_cfg$c python tools/profile_run.py > gpurun_out/ncup$c.log 2>&1
echo cfg$c rc=$?
ncu -i /tmp/r02p_cfg$c.ncu-rep --page raw --csv > gpurun_out/r02p_cfg${c}_raw.csv 2>&1
ncu -i /tmp/r02p_cfg$c.ncu-rep --page source --csv --print-source sass > gpurun_out/r02p_cfg${c}_src.csv 2>&1
ncu -i /tmp/r02p_cfg$c.ncu-rep --page details --csv > gpurun_out/r02p_cfg${c}_details.csv 2>&1
cp /tmp/r02p_cfg$c.ncu-rep gpurun_out/
done
du -sh gpurun_out
