#!/bin/bash
# Configs A and C and LOBPCG with the final build (parallel level-2 reduction)
cd "$GRAFT_REPO_ROOT"
timeout 1200 python tools/bench_configs.py A C > gpurun_out/r71_configs.jsonl 2> gpurun_out/r71_configs.err; echo "configs rc=$?"
cut -c1-600 gpurun_out/r71_configs.jsonl
timeout 900 python tools/bench_eigen.py 2d:1000 3d:128 > gpurun_out/r71_eigen.jsonl 2>&1; echo "eigen rc=$?"; cut -c1-400 gpurun_out/r71_eigen.jsonl | tail -3
