python tools/parity_diag.py 2 > gpurun_out/diag2.log 2>&1; echo rc=$?; cat gpurun_out/diag2.log
python tools/parity_diag.py 5 default simt > gpurun_out/diag5.log 2>&1; echo rc=$?; cat gpurun_out/diag5.log
python tools/parity_diag.py 3 default simt > gpurun_out/diag3.log 2>&1; echo rc=$?; cat gpurun_out/diag3.log
