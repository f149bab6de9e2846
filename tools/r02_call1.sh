set -x
nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
lscpu | grep -i "model name"
mem=$(free -g | awk '/Mem:/{print $2}')
if [ "$mem" -gt 150 ]; then
  nohup python tools/make_fullsize_golden.py --out gpurun_out/fullsize.json > gpurun_out/golden.log 2>&1 &
  GP=$!
fi
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
cat gpurun_out/bench1.json | head -c 600
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --plain-steps 0 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1; echo "ncu rc=$?"
if [ -n "$GP" ]; then wait $GP; fi
cat gpurun_out/golden.log
