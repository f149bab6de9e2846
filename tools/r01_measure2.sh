set -x
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q --timeout 600 2>&1 | tail -15
timeout 1200 python tools/bench_configs.py A C D E > gpurun_out/r01_configs.jsonl 2> gpurun_out/r01_configs.err; tail -3 gpurun_out/r01_configs.err; cut -c1-400 gpurun_out/r01_configs.jsonl
timeout 600 python bench.py --dist --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/r01_bench_dist1.json 2> gpurun_out/r01_bench_dist1.err; tail -3 gpurun_out/r01_bench_dist1.err; cat gpurun_out/r01_bench_dist1.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vec_kernel -s 3 -c 2 -o gpurun_out/r01_vec python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | tail -5
