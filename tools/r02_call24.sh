#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_xwin.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r61_xwin_pytest.log 2>&1; echo "xwin pytest rc=$?"
tail -2 gpurun_out/r61_xwin_pytest.log
timeout 1200 python tools/xw_sweep.py B D --variants=12,13 > gpurun_out/r61_xw_sweep.jsonl 2> gpurun_out/r61_xw_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r61_xw_sweep.jsonl"):
    d = json.loads(l)
    print(d["config"], d["setting"], d["xwin"]["variant"], d["xwin"].get("ctas_per_sm"), d["xwin"]["cap_x"], round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()})
PY
