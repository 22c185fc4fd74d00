for v in base fh6 fh7 base fh6 fh7; do KIFMM_LIB=variants/$v.so python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-100; done
