#!/bin/bash
# Round-1 final measurements on one B200: tests, smoke, bench (+reference arm), launch list,
# ncu captures, all configs, LOBPCG.
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/f_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 200 -c 40 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --plain-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_ws_kernel -s 3 -c 1 -o gpurun_out/f_spmv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --plain-steps 0 > /dev/null 2>&1
timeout 2400 python tools/bench_configs.py A C D D01 E > gpurun_out/f_configs.jsonl 2> gpurun_out/f_configs.err
timeout 900 python tools/bench_eigen.py 2d:1000 3d:128 > gpurun_out/f_eigen.jsonl 2>&1
grep -E "passed|failed" gpurun_out/f_pytest.log | tail -2; tail -1 gpurun_out/f_smoke.log; cut -c1-200 gpurun_out/f_bench.json; cut -c1-200 gpurun_out/f_bench_ref.json
