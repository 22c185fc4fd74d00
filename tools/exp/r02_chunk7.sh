KIFMM_LIB=variants/head.so python tools/exp/cmp_lib.py 5 save /tmp/ref5.npz
KIFMM_LIB=variants/head.so python tools/exp/cmp_lib.py 3 save /tmp/ref3.npz
for ch in 0 8; do KIFMM_FAR_CHUNK=$ch python tools/exp/cmp_lib.py 5 check /tmp/ref5.npz 2>&1 | tail -1; KIFMM_FAR_CHUNK=$ch python tools/exp/cmp_lib.py 3 check /tmp/ref3.npz 2>&1 | tail -1; done
for ch in 0 6 8 12 auto; do if [ $ch = auto ]; then unset KIFMM_FAR_CHUNK; else export KIFMM_FAR_CHUNK=$ch; fi
  echo "chunk $ch"; timeout 300 python tools/near_time.py 3 30 2>&1 | tail -1 | cut -c1-80; timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-80; done
unset KIFMM_FAR_CHUNK
timeout 900 python -m pytest tests/test_gpu_configs.py -q -k "3 or 5" -p no:cacheprovider 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu.py -q -k "parity_vs_oracle or sphere or two_cluster or queue or schedule" -p no:cacheprovider 2>&1 | tail -1
