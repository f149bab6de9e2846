#!/bin/bash
# Fixed-layout pair kernel + diagonal-warp BiCGStab SpMVs: full GPU suite, bench B/D/E,
# config B) and the launch list of the bench command.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r72_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r72_pytest.log | tail -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r72_smoke.log 2>&1; tail -1 gpurun_out/r72_smoke.log
timeout 900 python bench.py > gpurun_out/r72_benchB.json 2> gpurun_out/r72_benchB.err; echo "benchB rc=$?"
timeout 900 python bench.py --config D --no-cpu-baseline --plain-steps 50 > gpurun_out/r72_benchD.json 2> gpurun_out/r72_benchD.err; echo "benchD rc=$?"
timeout 900 python bench.py --config E --no-cpu-baseline --plain-steps 50 > gpurun_out/r72_benchE.json 2> gpurun_out/r72_benchE.err; echo "benchE rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r72_ref.json 2> gpurun_out/r72_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r72_launchesB.csv python bench.py --steps 3 --warmup 3 --plain-steps 0 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu B rc=$?"
for f in r72_benchB r72_benchD r72_benchE r72_ref; do cut -c1-250 gpurun_out/$f.json; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_dia -s 3 -c 1 -o gpurun_out/r72_diaD python tools/spmv_profile.py convdiff3d 368 bicgstab 0.1 > /dev/null 2>&1; echo "ncu diaD rc=$?"
