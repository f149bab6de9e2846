#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python tools/bench_eigen.py 2d:1000 3d:128 > gpurun_out/r14_eigen.jsonl 2>&1; echo "eig rc=$?"
cut -c1-500 gpurun_out/r14_eigen.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r14_eig_launches.csv python tools/eig_profile.py 1000 30 > gpurun_out/r14_eig_prof.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_kernel -s 10 -c 1 -o gpurun_out/r14_gram python tools/eig_profile.py 1000 10 > /dev/null 2>&1; echo "ncu gram rc=$?"
