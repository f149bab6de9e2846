#!/bin/bash
# Pattern-table SpMV: L2 prefetch distance sweep (SPARSLA_DIA_PREFETCH waves of resident CTAs)
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do for pf in 0 1 2 3; do
SPARSLA_DIA_PREFETCH=$pf timeout 300 python tools/spmv_profile.py poisson3d 464 cg 2>/dev/null | head -1 | sed "s/^/B pf=$pf /" | cut -c1-70
SPARSLA_DIA_PREFETCH=$pf timeout 300 python tools/spmv_profile.py convdiff3d 368 bicgstab 0.1 2>/dev/null | head -1 | sed "s/^/D pf=$pf /" | cut -c1-130
done; done
