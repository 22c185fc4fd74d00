timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gt1.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gt1.log
timeout 900 python tools/configs.py 2 3 5 > gpurun_out/configs235.jsonl 2> gpurun_out/configs.err; echo rc=$?
