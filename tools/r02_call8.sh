#!/bin/bash
# Round-2 measurement with the x-window SpMV default: GPU suite, smoke, bench B/D/E, configs
# A/C, launch list, ncu of the FEM x-window SpMV.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r8_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r8_pytest.log | tail -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r8_smoke.log 2>&1; tail -1 gpurun_out/r8_smoke.log
timeout 900 python bench.py > gpurun_out/r8_benchB.json 2> gpurun_out/r8_benchB.err; echo "benchB rc=$?"
timeout 900 python bench.py --config D --no-cpu-baseline --plain-steps 50 > gpurun_out/r8_benchD.json 2> gpurun_out/r8_benchD.err; echo "benchD rc=$?"
timeout 900 python bench.py --config E --no-cpu-baseline --plain-steps 50 > gpurun_out/r8_benchE.json 2> gpurun_out/r8_benchE.err; echo "benchE rc=$?"
timeout 1500 python tools/bench_configs.py A C > gpurun_out/r8_configs.jsonl 2> gpurun_out/r8_configs.err; echo "configs rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_xw_kernel -s 2 -c 1 -o gpurun_out/r8_fem_xw python tools/spmv_profile.py fem2d 4474 cg > /dev/null 2>&1; echo "ncu fem rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 100 -c 60 --csv --log-file gpurun_out/r8_launchesC.csv python tools/spmv_profile.py fem2d 4474 cg > /dev/null 2>&1; echo "ncu C rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r8_launchesB.csv python bench.py --steps 3 --warmup 3 --plain-steps 0 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu B rc=$?"
for f in r8_benchB r8_benchD r8_benchE; do cut -c1-200 gpurun_out/$f.json; done
cut -c1-300 gpurun_out/r8_configs.jsonl
