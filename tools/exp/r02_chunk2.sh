nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "5" -p no:cacheprovider 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -10
tail -1 gpurun_out/parity_r02.jsonl | cut -c1-400
for ch in 0 auto; do if [ $ch = auto ]; then unset KIFMM_FAR_CHUNK; else export KIFMM_FAR_CHUNK=$ch; fi; timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-300; done
unset KIFMM_FAR_CHUNK
KIFMM_LIB=variants/base.so timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-300
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv
