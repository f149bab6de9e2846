#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_gpu_dia.py tests/test_gpu_xwin.py tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider > gpurun_out/r71_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r71_pytest.log; grep -E "^FAILED" gpurun_out/r71_pytest.log | head
timeout 600 python tools/xw_sweep.py B E D > gpurun_out/r71_xw_sweep.jsonl 2>/dev/null; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r71_xw_sweep.jsonl"):
    d = json.loads(l)
    print(d["config"], d["setting"], d["xwin"]["variant"], d["dia"]["on"], round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()})
PY
