#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_gpu_xwin.py tests/test_gpu_dist.py tests/test_gpu_dist_ipc.py tests/test_gpu_torch_dist.py tests/test_gpu_bench.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r10_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r10_pytest.log | tail -8
timeout 900 python tools/spmv_longrow_bench.py 1000000 > gpurun_out/r10_longrow1m.jsonl 2>&1; echo "longrow1m rc=$?"
timeout 900 python tools/spmv_longrow_bench.py 4000000 > gpurun_out/r10_longrow4m.jsonl 2>&1; echo "longrow4m rc=$?"
cut -c1-600 gpurun_out/r10_longrow1m.jsonl gpurun_out/r10_longrow4m.jsonl
timeout 900 python bench.py --config D --no-cpu-baseline --plain-steps 50 > gpurun_out/r10_benchD.json 2> gpurun_out/r10_benchD.err; echo "benchD rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/r10_benchD.json').read().strip().splitlines()[-1])
print(json.dumps({k: d[k] for k in ('value','kernel_ms','roofline','format','plain_csr','plain_values_xwin')})[:3000])
"
