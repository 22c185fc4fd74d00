# A/B of node-local geometry in check / far kernels: parity vs oracle at configs 2, 3, 5
for v in lc0lf0 lc1lf0 lc0lf1 default; do
  if [ $v = default ]; then unset KIFMM_LIB; else export KIFMM_LIB=variants/$v.so; fi
  rm -f gpurun_out/parity_r02.jsonl
  timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider -k "2 or 3 or 5" 2>&1 | tail -1
  python - <<P
import json
for l in open('gpurun_out/parity_r02.jsonl'):
    c=json.loads(l); print("$v", c["config"], "%.3e"%c["rel_l2_potential_vs_oracle"], "%.3e"%c["rel_l2_potential_vs_direct_1000"])
P
done
