#!/bin/bash
# A/B inside bench.py (config B): parallel level-2 reduction on/off, far diagonals without L1 allocation
cd "$GRAFT_REPO_ROOT"
SPARSLA_DIA_VARIANT=14 timeout 600 python -m pytest tests/test_gpu_dia.py -q --timeout 300 -p no:cacheprovider > gpurun_out/r74_pytest.log 2>&1; echo "pytest v14 rc=$?"; tail -1 gpurun_out/r74_pytest.log
for rep in 1 2; do
for cfg in "SPARSLA_MULTI_FINISH=0" "SPARSLA_MULTI_FINISH=1" "SPARSLA_DIA_VARIANT=14" "SPARSLA_DIA_VARIANT=15"; do
env $cfg timeout 600 python bench.py --plain-steps 0 --no-cpu-baseline --e2e-steps 1 --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value'],1), {k: round(v,4) for k,v in d['kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done; done
