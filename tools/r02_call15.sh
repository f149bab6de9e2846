#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_eigen.py tests/test_gpu_torch.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r15_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r15_pytest.log | tail -5
for g in 0 1; do SPARSLA_GRAM_WS=$g timeout 900 python tools/bench_eigen.py 2d:1000 3d:128 2>&1 | cut -c1-260 | sed "s/^/gram_ws=$g /"; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r15_eig_launches.csv python tools/eig_profile.py 1000 30 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_ws_kernel -s 10 -c 2 -o gpurun_out/r15_gramws python tools/eig_profile.py 1000 10 > /dev/null 2>&1; echo "ncu gram rc=$?"
