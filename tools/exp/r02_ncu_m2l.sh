# ncu --set full of the tcgen05 M2L kernel: config 2 (row width 160, 2-CTA pair) and config 1 (row width 128)
set -x
mkdir -p gpurun_out
for c in 2 1; do
KIFMM_CFG=$c KIFMM_ITERS=1 timeout 600 python tools/profile_run.py > gpurun_out/pm$c.log 2>&1 && \
KIFMM_CFG=$c KIFMM_ITERS=1 timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"m2l_tc_kernel|m2l_tc_reduce" -c 14 -o /tmp/r02_m2l_cfg$c python tools/profile_run.py > gpurun_out/ncum$c.log 2>&1
echo cfg$c rc=$?
ncu -i /tmp/r02_m2l_cfg$c.ncu-rep --page raw --csv > gpurun_out/r02_ncu_raw_cfg${c}_m2l.csv 2>&1
done
ls -la gpurun_out | tail -5
