#!/bin/bash
# Round-2 closing check (driver-like): : full GPU suite, smoke, bench B/D/E + reference arm, ncu, launch list
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r77_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r77_pytest.log | tail -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r77_smoke.log 2>&1; tail -1 gpurun_out/r77_smoke.log
timeout 900 python bench.py > gpurun_out/r77_benchB.json 2> gpurun_out/r77_benchB.err; echo "benchB rc=$?"
timeout 900 python bench.py --config D --no-cpu-baseline --plain-steps 50 > gpurun_out/r77_benchD.json 2> gpurun_out/r77_benchD.err; echo "benchD rc=$?"
timeout 900 python bench.py --config E --no-cpu-baseline --plain-steps 50 > gpurun_out/r77_benchE.json 2> gpurun_out/r77_benchE.err; echo "benchE rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r77_ref.json 2> gpurun_out/r77_ref.err; echo "ref rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_diac_kernel -s 3 -c 1 -o gpurun_out/r77_diacB python bench.py --steps 3 --warmup 3 --plain-steps 0 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu dia rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r77_launchesB.csv python bench.py --steps 3 --warmup 3 --plain-steps 0 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu B rc=$?"
for f in r77_benchB r77_benchD r77_benchE r77_ref; do cut -c1-300 gpurun_out/$f.json; done
