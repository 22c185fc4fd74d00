rm -f gpurun_out/ozaki_r02.jsonl
timeout 900 python -m pytest tests/test_gpu.py -q -k "ozaki or int8 or fp64" -p no:cacheprovider 2>&1 | tail -1
cat gpurun_out/ozaki_r02.jsonl | cut -c1-200
timeout 600 python tools/near_time.py 4 5 2>&1 | tail -1 | cut -c1-400
KIFMM_CFG=4 KIFMM_ITERS=1 timeout 900 ncu -f --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:"m2l_oz_kernel" -c 1 python tools/profile_run.py 2>&1 | grep -E "m2l_oz|duration|bytes|throughput|tensor" | head
