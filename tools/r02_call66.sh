#!/bin/bash
# Pattern-table diagonal kernel (spmv_diac_kernel, variants 6..8): parity, sweep, ncu.
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_dia.py -q --timeout 300 -p no:cacheprovider > gpurun_out/r66_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r66_pytest.log
SPARSLA_DIA_VARIANT=12 timeout 900 python -m pytest tests/test_gpu_dia.py -q --timeout 300 -p no:cacheprovider > gpurun_out/r66_pytest3.log 2>&1; echo "pytest v3 rc=$?"; tail -1 gpurun_out/r66_pytest3.log
grep -E "^FAILED|Error" gpurun_out/r66_pytest.log gpurun_out/r66_pytest3.log | head -10
for v in 7 12 13; do
SPARSLA_DIA_VARIANT=$v timeout 300 python tools/spmv_profile.py poisson3d 464 cg 2>/dev/null | head -1 | sed "s/^/B v=$v /" | cut -c1-120
SPARSLA_DIA_VARIANT=$v timeout 300 python tools/spmv_profile.py convdiff3d 368 bicgstab 0.1 2>/dev/null | head -1 | sed "s/^/D v=$v /" | cut -c1-200
done
SPARSLA_DIA_VARIANT=12 timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_diac_kernel -s 3 -c 1 -o gpurun_out/r66_diac python tools/spmv_profile.py poisson3d 464 cg > /dev/null 2>&1; echo "ncu rc=$?"
