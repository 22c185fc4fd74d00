timeout 900 python -m pytest tests/test_gpu.py -q -k "parity_vs_oracle or queue_mode or schedule or tiny or coincident or small_trees" -p no:cacheprovider 2>&1 | tail -1
for c in 2 3; do python tools/exp/cmp_lib.py $c check /tmp/none.npz 2>/dev/null | tail -0; done
KIFMM_LIB=variants/base.so python tools/exp/cmp_lib.py 3 save /tmp/ref3.npz; python tools/exp/cmp_lib.py 3 check /tmp/ref3.npz 2>&1 | tail -1
for ch in 0 8 16; do KIFMM_FAR_CHUNK=$ch timeout 300 python tools/near_time.py 3 30 2>&1 | tail -1 | cut -c1-90; done
timeout 300 python tools/near_time.py 3 30 2>&1 | tail -1 | cut -c1-90
KIFMM_FAR_CHUNK=0 timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-90
timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-90
timeout 900 python -m pytest tests/test_gpu_configs.py -q -k "3 or 5" -p no:cacheprovider 2>&1 | tail -1
tail -2 gpurun_out/parity_r02.jsonl | cut -c1-260
