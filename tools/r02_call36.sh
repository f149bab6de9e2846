#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_eigen.py tests/test_gpu_torch.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r36_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed|Error" gpurun_out/r36_pytest.log | tail -12
for dv in 0 1; do SPARSLA_EIG_DEVICE=$dv timeout 900 python tools/bench_eigen.py 2d:1000 3d:128 2>&1 | cut -c1-330 | sed "s/^/device=$dv /"; done
