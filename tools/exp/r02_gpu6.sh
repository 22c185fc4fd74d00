timeout 900 python -m pytest tests/test_gpu.py -q -x -k "parity_vs_oracle or config2 or queue or schedule or evaluate_many" > gpurun_out/t6.log 2>&1; echo t rc=$?; tail -2 gpurun_out/t6.log
rm -f gpurun_out/parity_r02.jsonl
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x > gpurun_out/t6c.log 2>&1; echo tc rc=$?; tail -2 gpurun_out/t6c.log
for v in default u8 minb8 minb10; do
  if [ $v = default ]; then L=""; else L="variants/$v.so"; fi
  KIFMM_LIB=$L KIFMM_NEAR_BPS=0 python tools/near_time.py 2 30 2>&1 | tail -1
done
python tools/near_time.py 5 5 2>&1 | tail -1
python tools/near_time.py 3 20 2>&1 | tail -1
