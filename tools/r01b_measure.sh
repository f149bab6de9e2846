#!/bin/bash
# Round-1b measurements on one B200: launch list + ncu full captures of the CG kernels, all configs, LOBPCG.
cd "$GRAFT_REPO_ROOT"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/r01b_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --plain-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_ws_kernel -s 3 -c 1 -o gpurun_out/r01b_spmv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --plain-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vec_kernel -s 3 -c 2 -o gpurun_out/r01b_vec python bench.py --steps 5 --warmup 3 --no-cpu-baseline --plain-steps 0 > /dev/null 2>&1
timeout 2400 python tools/bench_configs.py A C D D01 E > gpurun_out/r01b_configs.jsonl 2> gpurun_out/r01b_configs.err
timeout 900 python tools/bench_eigen.py 2d:1000 3d:128 > gpurun_out/r01b_eigen.jsonl 2>&1
ls -la gpurun_out/ | tail -12
