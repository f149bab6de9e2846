# A/B of the fused small-problem CG kernel (config A): resident chunk images on / off
run() { timeout 300 python tools/bench_configs.py A 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['iterations'], round(d['time_to_tolerance_s']*1e3,2), round(d['kernel_ms']['spmv_cg']*1e3,2))"; }
for rep in 1 2 3; do
SPARSLA_FUSED_RESIDENT=0 run off
run resident
done
