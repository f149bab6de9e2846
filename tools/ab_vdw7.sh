# Dictionary-kernel variants on config B (SPARSLA_VD_VARIANT): 0 = 8-wide 3 CTAs/SM,
# 3 = 7-wide 4 CTAs/SM (default for rows <= 7), 4 = 7-wide 3 CTAs/SM
for rep in 1 2; do for v in 0 3 4; do
SPARSLA_VD_VARIANT=$v timeout 600 python bench.py --no-cpu-baseline --plain-steps 0 --steps 100 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('vd=$v', round(d['value'],1), {k: round(x*1e3,1) for k,x in d['kernel_ms'].items()}, d['parity_gate']['ok'])"
done; done
