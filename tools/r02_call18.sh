#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for pol in 0 1 2; do
  SPARSLA_XW_XPOL=$pol timeout 600 python tools/xw_sweep.py B 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['setting'] in ('xwin-1',): print('xpol=$pol', d['setting'], round(d['ms']['spmv_cg'],4))
"
  SPARSLA_XW_XPOL=$pol timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:spmv_xw -s 3 -c 2 --csv python tools/spmv_profile.py poisson3d 464 cg 2>/dev/null | grep spmv_xw | awk -F'","' '{print "xpol='$pol' " $(NF-2) " " $NF}'
done
