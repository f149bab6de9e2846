#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "long_rows or hub or direct" --timeout 600 -p no:cacheprovider > gpurun_out/r11_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r11_pytest.log | tail -8
timeout 900 python tools/spmv_longrow_bench.py 1000000 > gpurun_out/r11_longrow1m.jsonl 2>&1; echo "longrow1m rc=$?"
timeout 900 python tools/spmv_longrow_bench.py 4000000 > gpurun_out/r11_longrow4m.jsonl 2>&1; echo "longrow4m rc=$?"
cut -c1-420 gpurun_out/r11_longrow1m.jsonl gpurun_out/r11_longrow4m.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r11_longrow_launches.csv python tools/spmv_longrow_bench.py 4000000 > /dev/null 2>&1; echo "ncu rc=$?"
