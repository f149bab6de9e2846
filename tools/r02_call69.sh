#!/bin/bash
# Parallel level-2 reduction restricted to single-launch, non-peer points: full GPU suite + bench B/D/E
cd "$GRAFT_REPO_ROOT"
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r69_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r69_pytest.log | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r69_smoke.log 2>&1; tail -1 gpurun_out/r69_smoke.log
timeout 900 python bench.py > gpurun_out/r69_benchB.json 2> gpurun_out/r69_benchB.err; echo "benchB rc=$?"
timeout 900 python bench.py --config D --no-cpu-baseline --plain-steps 50 > gpurun_out/r69_benchD.json 2> gpurun_out/r69_benchD.err; echo "benchD rc=$?"
timeout 900 python bench.py --config E --no-cpu-baseline --plain-steps 50 > gpurun_out/r69_benchE.json 2> gpurun_out/r69_benchE.err; echo "benchE rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r69_launchesB.csv python bench.py --steps 3 --warmup 3 --plain-steps 0 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu B rc=$?"
for f in r69_benchB r69_benchD r69_benchE; do cut -c1-200 gpurun_out/$f.json; done
