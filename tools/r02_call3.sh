#!/bin/bash
# Round-2: x-window SpMV parity + A/B sweep, then the full GPU suite.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python -m pytest tests/test_gpu_xwin.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r3_xwin_pytest.log 2>&1; echo "xwin pytest rc=$?"
tail -3 gpurun_out/r3_xwin_pytest.log
timeout 1200 python tools/xw_sweep.py B E D C --variants=0,1,2,3,4,5 > gpurun_out/r3_xw_sweep.jsonl 2> gpurun_out/r3_xw_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r3_xw_sweep.jsonl"):
    d = json.loads(l)
    print(d["config"], d["setting"], d["xwin"]["variant"], round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()}, {k: round(v, 3) for k, v in d.items() if k.endswith("_frac")})
PY
tail -5 gpurun_out/r3_xw_sweep.err
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r3_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r3_pytest.log | tail -30
