#!/bin/bash
# Vector kernels: resident (persistent) grid vs one chunk per CTA, with the parallel level-2 reduction
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do for vp in 0 1; do
SPARSLA_VEC_PERSIST=$vp timeout 600 python bench.py --plain-steps 0 --no-cpu-baseline --e2e-steps 1 --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B persist=$vp', round(d['value'],1), {k: round(v,4) for k,v in d['kernel_ms'].items()}, d['parity_gate']['ok'])"
SPARSLA_VEC_PERSIST=$vp timeout 300 python tools/spmv_profile.py convdiff3d 368 bicgstab 0.1 2>/dev/null | head -1 | sed "s/^/D persist=$vp /" | cut -c1-200
done; done
