#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_xwin.py tests/test_gpu_dist.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r34_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r34_pytest.log | tail -3
timeout 600 python tools/vec_ab.py 2>&1 | head -1
timeout 1200 python tools/xw_sweep.py B E D > gpurun_out/r34_xw_sweep.jsonl 2> gpurun_out/r34_xw_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r34_xw_sweep.jsonl"):
    d = json.loads(l)
    if "plain" in d["setting"]: continue
    print(d["config"], d["setting"], d["xwin"]["variant"], round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()})
PY
