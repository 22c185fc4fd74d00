timeout 1500 python -m pytest tests/test_gpu_configs.py -m gpu -q -s > gpurun_out/gputests_cfg.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gputests_cfg.log
