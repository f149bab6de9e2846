NVAR=7 python tools/spmv_sweep.py fem2d 4474 2601 2>&1 | cut -c1-130
for g in 2 4 8; do echo "U1 group $g"; SPARSLA_U1_GROUP=$g NVAR=1 python tools/spmv_sweep.py poisson3d 464 2>&1 | cut -c1-160; done
for k in 0 1; do echo "L2_KEEP=$k"; SPARSLA_L2_KEEP=$k python tools/bench_configs.py A 2>&1 | cut -c1-420; done
