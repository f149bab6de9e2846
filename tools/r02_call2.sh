#!/bin/bash
# Round-2 measurement pass: GPU tests (incl. full-size golden gates), bench B/D/E, long-row
# SpMV, launch list, ncu capture of the BiCGStab t-SpMV (config D').
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|error" gpurun_out/r2_pytest.log | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; tail -1 gpurun_out/r2_smoke.log
timeout 900 python bench.py > gpurun_out/r2_benchB.json 2> gpurun_out/r2_benchB.err; echo "benchB rc=$?"
timeout 900 python bench.py --config D --no-cpu-baseline --plain-steps 50 > gpurun_out/r2_benchD.json 2> gpurun_out/r2_benchD.err; echo "benchD rc=$?"
SPARSLA_BICGT_VD7=1 timeout 900 python bench.py --config D --no-cpu-baseline --plain-steps 0 > gpurun_out/r2_benchD7.json 2> gpurun_out/r2_benchD7.err; echo "benchD7 rc=$?"
timeout 900 python bench.py --config E --no-cpu-baseline --plain-steps 50 > gpurun_out/r2_benchE.json 2> gpurun_out/r2_benchE.err; echo "benchE rc=$?"
timeout 600 python tools/spmv_longrow_bench.py > gpurun_out/r2_longrow.jsonl 2>&1; echo "longrow rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 100 -c 60 --csv --log-file gpurun_out/r2_launchesD.csv python tools/spmv_profile.py convdiff3d 368 bicgstab 0.1 > /dev/null 2>&1; echo "ncu D rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:spmv_ws_kernelILi3E -s 2 -c 1 -o gpurun_out/r2_spmvT python tools/spmv_profile.py convdiff3d 368 bicgstab 0.1 > /dev/null 2>&1; echo "ncu T rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launchesB.csv python bench.py --steps 3 --warmup 3 --plain-steps 0 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu B rc=$?"
for f in r2_benchB r2_benchD r2_benchD7 r2_benchE; do cut -c1-300 gpurun_out/$f.json; done
cat gpurun_out/r2_longrow.jsonl | cut -c1-400
