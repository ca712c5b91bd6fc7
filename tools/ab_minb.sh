mkdir -p gpurun_out
python bench.py --no-cpu-baseline > gpurun_out/ab_minb5.log 2>&1
(cd paper_2111_01083_b200 && touch csrc/cuda/near_sym.cu && make EXTRA_NVFLAGS=-DPWB_SYM_LAPLACE_MINB=6 > /dev/null 2>&1)
python bench.py --no-cpu-baseline > gpurun_out/ab_minb6.log 2>&1
for f in gpurun_out/ab_*.log; do python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('$f', round(r['near_ms_per_launch'],2), round(r['fp64_pipe_frac'],4))
"; done
