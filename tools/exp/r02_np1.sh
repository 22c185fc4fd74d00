# tcgen05 path for p = 4, 5 (row widths 64, 128): parity tests and config 1 timing
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -rf -p no:cacheprovider -k "parity_vs_oracle or tcgen05 or scheduling or smoke or small" > gpurun_out/np1_tests.log 2>&1; echo rc=$?; tail -15 gpurun_out/np1_tests.log
timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -rf -p no:cacheprovider -k "1 or 2" > gpurun_out/np1_cfg.log 2>&1; echo rc=$?; tail -5 gpurun_out/np1_cfg.log
timeout 600 python tools/configs.py 1 2 > gpurun_out/np1_configs.jsonl 2> gpurun_out/np1_configs.err; echo rc=$?; cut -c1-400 gpurun_out/np1_configs.jsonl
