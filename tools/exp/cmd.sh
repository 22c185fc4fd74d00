timeout 1200 python tools/configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo configs rc=$?
bash tools/exp/final.sh
