#!/bin/bash
# diagonal-warp SpMV: tests + sweep against the x-window / gather kernels
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_dia.py -q --timeout 300 -p no:cacheprovider > gpurun_out/r68_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r68_pytest.log; grep -E "^FAILED|Error" gpurun_out/r68_pytest.log | head -20
timeout 900 python tools/xw_sweep.py B E D > gpurun_out/r68_xw_sweep.jsonl 2> gpurun_out/r68_xw_sweep.err; echo "sweep rc=$?"; tail -3 gpurun_out/r68_xw_sweep.err
python - <<'PY'
import json
for l in open("gpurun_out/r68_xw_sweep.jsonl"):
    d = json.loads(l)
    print(d["config"], d["setting"], d["xwin"]["variant"], d["dia"], round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()})
PY
