# 7-wide dictionary kernel at 4 CTAs/SM (default for rows <= 7) vs the 8-wide 3-CTA kernel
for rep in 1 2; do for v in 0 3; do
SPARSLA_VD_VARIANT=$v timeout 600 python tools/bench_configs.py D E 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('vd=$v', d['config'][:3], d['iterations'], round(d['it_per_s'],1), {k: round(x*1e3,1) for k,x in d['kernel_ms'].items()})"
done; done
