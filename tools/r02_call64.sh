#!/bin/bash
# dia info ABI (pattern count), bench roofline (dominant kernel + SpMV sub-object), bench tests
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_gpu_dia.py tests/test_gpu_bench.py tests/test_gpu_xwin.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r64_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r64_pytest.log
grep -E "^FAILED|Error" gpurun_out/r64_pytest.log | head
timeout 900 python bench.py --plain-steps 0 --no-cpu-baseline > gpurun_out/r64_benchB.json 2> gpurun_out/r64_benchB.err; echo "benchB rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r64_benchB.json')); print(d['value'], json.dumps(d['roofline']))"
