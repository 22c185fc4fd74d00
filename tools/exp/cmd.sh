timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gt1.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gt1.log
for i in 1 2; do python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-100; KIFMM_TC_FACE=0 python tools/near_time.py 2 40 2>&1 | tail -1 | cut -c1-100; done
python -c "
import sys; sys.path.insert(0,'.')
from paper_2303_08394_b200 import fmm, generators
c=generators.CONFIGS[2]; pos,q=generators.config_sample(2)
f=fmm.Fmm(pos, fmm.FmmConfig(p=6,n_crit=150,precision=32,gradient=True)); i=f.info(); print('slots', i['m2l_pairs'], i['m2l_padded_pairs'])"
