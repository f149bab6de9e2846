#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "long_rows or hub or direct" --timeout 600 -p no:cacheprovider > gpurun_out/r12_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r12_pytest.log | tail -8
for t in auto 16 32 64; do
  if [ $t = auto ]; then unset SPARSLA_LONG_ROW; else export SPARSLA_LONG_ROW=$t; fi
  timeout 900 python tools/spmv_longrow_bench.py 4000000 2>&1 | head -1 | cut -c1-330 | sed "s/^/thr=$t /"
done
unset SPARSLA_LONG_ROW
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r12_longrow_launches.csv python tools/spmv_longrow_bench.py 4000000 > /dev/null 2>&1; echo "ncu rc=$?"
