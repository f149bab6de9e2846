#!/bin/bash
# Speculative round-0 loads (variants 16, 17) vs default 7: parity + bench A/B (config B, D')
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_dia.py -q --timeout 300 -p no:cacheprovider > gpurun_out/r76_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r76_pytest.log
SPARSLA_DIA_VARIANT=16 timeout 600 python -m pytest tests/test_gpu_dia.py -q --timeout 300 -p no:cacheprovider > gpurun_out/r76_pytest16.log 2>&1; echo "pytest v16 rc=$?"; tail -1 gpurun_out/r76_pytest16.log
for rep in 1 2; do
for v in 7 16 17; do
SPARSLA_DIA_VARIANT=$v timeout 600 python bench.py --plain-steps 0 --no-cpu-baseline --e2e-steps 1 --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('B v=$v', round(d['value'],1), {k: round(v,4) for k,v in d['kernel_ms'].items()}, d['clocks']['sm_mhz'])"
SPARSLA_DIA_VARIANT=$v timeout 300 python tools/spmv_profile.py convdiff3d 368 bicgstab 0.1 2>/dev/null | head -1 | sed "s/^/D v=$v /" | cut -c1-130
done; done
