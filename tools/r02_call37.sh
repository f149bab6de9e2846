#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_dia.py -q --timeout 300 -p no:cacheprovider > gpurun_out/r74_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r74_pytest.log
timeout 600 python tools/xw_sweep.py B D > gpurun_out/r74_xw_sweep.jsonl 2>/dev/null; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r74_xw_sweep.jsonl"):
    d = json.loads(l)
    if "plain" not in d["setting"]:
        print(d["config"], d["setting"], d["dia"]["modes"], round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()})
PY
