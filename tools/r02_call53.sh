#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/r53_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r53_pytest.log | tail -5
timeout 1200 python tools/xw_sweep.py B E > gpurun_out/r53_xw_sweep.jsonl 2> gpurun_out/r53_xw_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r53_xw_sweep.jsonl"):
    d = json.loads(l)
    if "plain" in d["setting"]: continue
    print(d["config"], d["setting"], d["xwin"]["variant"], round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()})
PY
