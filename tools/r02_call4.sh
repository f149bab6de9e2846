#!/bin/bash
# x-window SpMV diagnosis: ncu --set full of the x-window and the gather dictionary kernels (config E).
cd "$GRAFT_REPO_ROOT"
SPARSLA_XWIN=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_xw_kernel -s 2 -c 1 -o gpurun_out/r4_xw python tools/spmv_profile.py poisson3d 368 cg > gpurun_out/r4_xw.log 2>&1; echo "ncu xw rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_ws_kernel -s 2 -c 1 -o gpurun_out/r4_ws python tools/spmv_profile.py poisson3d 368 cg > gpurun_out/r4_ws.log 2>&1; echo "ncu ws rc=$?"
timeout 900 python -m pytest tests/test_gpu_xwin.py -q --timeout 300 -p no:cacheprovider > gpurun_out/r4_xwin_pytest.log 2>&1; echo "xwin pytest rc=$?"
tail -3 gpurun_out/r4_xwin_pytest.log
