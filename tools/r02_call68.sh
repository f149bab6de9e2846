#!/bin/bash
# Parallel level-2 reduction (multi_finish): full GPU suite, A/B of the kernel times
cd "$GRAFT_REPO_ROOT"
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/r68_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r68_pytest.log | tail -5
for rep in 1 2; do for mf in 0 1; do
SPARSLA_MULTI_FINISH=$mf timeout 300 python tools/spmv_profile.py poisson3d 464 cg 2>/dev/null | head -1 | sed "s/^/B mf=$mf /" | cut -c1-130
SPARSLA_MULTI_FINISH=$mf timeout 300 python tools/spmv_profile.py convdiff3d 368 bicgstab 0.1 2>/dev/null | head -1 | sed "s/^/D mf=$mf /" | cut -c1-210
done; done
