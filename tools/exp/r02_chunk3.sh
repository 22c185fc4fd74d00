for lib in default variants/nopf.so variants/base.so; do
  echo "== $lib"
  if [ $lib != default ]; then export KIFMM_LIB=$lib; else unset KIFMM_LIB; fi
  timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "5 or 3" -p no:cacheprovider 2>&1 | tail -1
  KIFMM_FAR_CHUNK=0 timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-100
  timeout 300 python tools/near_time.py 5 3 2>&1 | tail -1 | cut -c1-100
  timeout 300 python tools/near_time.py 3 30 2>&1 | tail -1 | cut -c1-100
done
