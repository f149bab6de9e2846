#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_eigen.py tests/test_gpu_torch.py tests/test_cpp_dropin.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r32_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r32_pytest.log | tail -5
SPARSLA_EIG_TIMING=1 timeout 900 python tools/bench_eigen.py 2d:1000 3d:128 2>&1 | cut -c1-330
