timeout 900 python -m pytest tests/test_gpu.py -q -x -k "parity_vs_oracle or config2 or queue or evaluate_many or small_trees or tiny or coincident" > gpurun_out/t7.log 2>&1; echo t rc=$?; tail -3 gpurun_out/t7.log
rm -f gpurun_out/parity_r02.jsonl
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x > gpurun_out/t7c.log 2>&1; echo tc rc=$?; tail -2 gpurun_out/t7c.log
for w in 1 0; do for b in 0 2; do
  echo "NEAR_WARP=$w BPS=$b"; KIFMM_NEAR_WARP=$w KIFMM_NEAR_BPS=$b python tools/near_time.py 2 30 2>&1 | tail -1
done; done
for w in 1 0; do KIFMM_NEAR_WARP=$w python tools/near_time.py 3 20 2>&1 | tail -1; KIFMM_NEAR_WARP=$w python tools/near_time.py 5 3 2>&1 | tail -1; done
