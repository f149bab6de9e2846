timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x --timeout 600 -k config_C 2>&1 | grep -E "assert|Error|passed|failed" | head -20
timeout 1500 python tools/bench_configs.py D D01 > gpurun_out/r01_configs_D.jsonl 2> gpurun_out/r01_configs_D.err; tail -3 gpurun_out/r01_configs_D.err; cut -c1-600 gpurun_out/r01_configs_D.jsonl
