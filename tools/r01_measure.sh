set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
lscpu | grep -E "Model name|^CPU\(s\)"
timeout 900 python -m pytest tests/ -m gpu -q --timeout 300 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err; tail -2 gpurun_out/r01_bench.err; cat gpurun_out/r01_bench.json
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r01_bench_ref.json 2> gpurun_out/r01_bench_ref.err; cat gpurun_out/r01_bench_ref.json
timeout 600 python bench.py --dist --steps 50 --warmup 3 --size 256 --no-cpu-baseline > gpurun_out/r01_bench_dist1.json 2> gpurun_out/r01_bench_dist1.err; tail -3 gpurun_out/r01_bench_dist1.err; cat gpurun_out/r01_bench_dist1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_ws_kernel -s 3 -c 1 -o gpurun_out/r01_spmv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:vec_kernel<1>" -s 2 -c 1 -o gpurun_out/r01_cgu1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:vec_kernel<2>" -s 2 -c 1 -o gpurun_out/r01_cgu2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
