#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for v in 0 1 2 4; do for pf in 1 2; do
SPARSLA_DIA_VARIANT=$v SPARSLA_DIA_PREFETCH=$pf timeout 300 python tools/spmv_profile.py poisson3d 464 cg 2>/dev/null | head -1 | sed "s/^/v=$v pf=$pf /" | cut -c1-60
done; done
SPARSLA_DIA=0 timeout 300 python tools/spmv_profile.py poisson3d 464 cg 2>/dev/null | head -1 | sed "s/^/xw /" | cut -c1-60
