# ncu --set full of the P2P kernels after the node-local geometry change (configs 2, 3, 5; near field standalone)
set -x
mkdir -p gpurun_out
for c in 2 3 5; do
KIFMM_NEAR_BPS=0 KIFMM_CFG=$c KIFMM_ITERS=1 timeout 600 python tools/profile_run.py > gpurun_out/pf$c.log 2>&1 && \
KIFMM_NEAR_BPS=0 KIFMM_CFG=$c KIFMM_ITERS=1 timeout 1500 ncu -f --set full --clock-control none \
  -k regex:"leaf_eval|far_hw|far_f2|check_f2|check_hw" -c 5 -o /tmp/r02f_cfg$c python tools/profile_run.py > gpurun_out/ncuf$c.log 2>&1
echo cfg$c rc=$?
ncu -i /tmp/r02f_cfg$c.ncu-rep --page raw --csv > gpurun_out/r02_ncu_raw_cfg${c}_p2p_final.csv 2>&1
done
ls -la gpurun_out | tail -4
