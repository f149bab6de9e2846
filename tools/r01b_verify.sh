#!/bin/bash
# Round-1 (session 2) verification on a B200: GPU tests, smoke, default bench.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v_gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/v_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/v_smoke.log
timeout 900 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo "bench exit $?" >> gpurun_out/v_bench.err
grep -E "passed|failed|^E |FAILED" gpurun_out/v_pytest.log | head -20; tail -2 gpurun_out/v_smoke.log; cut -c1-600 gpurun_out/v_bench.json; tail -3 gpurun_out/v_bench.err
