python tools/parity_diag.py 2 default simt > gpurun_out/diag2b.log 2>&1; echo rc=$?; cat gpurun_out/diag2b.log
python tools/parity_diag.py 5 default > gpurun_out/diag5b.log 2>&1; echo rc=$?; cat gpurun_out/diag5b.log
for i in 1 2; do python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/b5.log 2>&1; tail -1 gpurun_out/b5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms'])"; done
rm -f gpurun_out/parity_r02.jsonl
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu.py -q -x -k "config or tcgen05 or simt_gemms or schedule" > gpurun_out/t5.log 2>&1; echo t rc=$?; tail -3 gpurun_out/t5.log
