#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_dia -s 3 -c 1 -o gpurun_out/r67_diaB python tools/spmv_profile.py poisson3d 464 cg > /dev/null 2>&1; echo "ncu dia rc=$?"
