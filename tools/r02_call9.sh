#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_xwin.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r9_xwin_pytest.log 2>&1; echo "xwin pytest rc=$?"
tail -3 gpurun_out/r9_xwin_pytest.log
timeout 1200 python tools/xw_sweep.py B E D --variants=0,6,7,8 > gpurun_out/r9_xw_sweep.jsonl 2> gpurun_out/r9_xw_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r9_xw_sweep.jsonl"):
    d = json.loads(l)
    print(d["config"], d["setting"], d["xwin"]["variant"], d["xwin"]["modes"], round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()})
PY
tail -3 gpurun_out/r9_xw_sweep.err
SPARSLA_XW_VARIANT=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_xw_kernel -s 2 -c 1 -o gpurun_out/r9_pair python tools/spmv_profile.py poisson3d 464 cg > /dev/null 2>&1; echo "ncu pair rc=$?"
