#!/bin/bash
# diagonal-warp stream (value stream 3) vs pair: B sweep + one ncu --set full capture each
cd "$GRAFT_REPO_ROOT"
timeout 600 python tools/xw_sweep.py B --variants=12 > gpurun_out/r63_xw_sweep.jsonl 2> gpurun_out/r63_xw_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r63_xw_sweep.jsonl"):
    d = json.loads(l)
    print(d["config"], d["setting"], d["xwin"]["variant"], d["xwin"].get("diag_warps"), round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()})
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_xw -s 3 -c 1 -o gpurun_out/r63_dwB python tools/spmv_profile.py poisson3d 464 cg > /dev/null 2>&1; echo "ncu dw rc=$?"
SPARSLA_XW_DW=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_xw -s 3 -c 1 -o gpurun_out/r63_pairB python tools/spmv_profile.py poisson3d 464 cg > /dev/null 2>&1; echo "ncu pair rc=$?"
