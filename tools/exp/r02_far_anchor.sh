rm -f gpurun_out/parity_r02.jsonl
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider -k "2 or 3 or 5" 2>&1 | tail -1
python - <<P
import json
for l in open('gpurun_out/parity_r02.jsonl'):
    c=json.loads(l); print("anchor", c["config"], "%.3e"%c["rel_l2_potential_vs_oracle"], c.get("rel_l2_gradient_vs_oracle"))
P
python tools/exp/r02_deep.py 2>&1 | tail -5 | cut -c1-200
python tools/configs.py 2 3 5 | python -c "
import sys,json
for l in sys.stdin:
    c=json.loads(l); print(c['config'], round(c['eval_ms_median'],3), round(c['eval_ms_min'],3), c['phases_serialized_ms']['leaf_ms'])
"
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -p no:cacheprovider -k "deep or degenerate or far_surface or scaled or parity_vs_oracle or no_state" 2>&1 | tail -2
