cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_eigen.py tests/test_gpu_torch.py tests/test_cpp_dropin.py -q 2>&1 | grep -E "assert|Error|passed|failed" | head -20
timeout 900 python tools/bench_eigen.py 2d:1000 3d:128 2>&1 | tail -5
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/eig_launches.csv python tools/eig_profile.py 1000 30 > gpurun_out/eig_prof.log 2>&1; tail -1 gpurun_out/eig_prof.log
