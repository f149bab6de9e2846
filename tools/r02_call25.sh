#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_xwin.py -q --timeout 300 -p no:cacheprovider > gpurun_out/r62_xwin_pytest.log 2>&1; echo "xwin pytest rc=$?"
tail -2 gpurun_out/r62_xwin_pytest.log
timeout 1200 python tools/xw_sweep.py B E D C --variants=12 > gpurun_out/r62_xw_sweep.jsonl 2> gpurun_out/r62_xw_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r62_xw_sweep.jsonl"):
    d = json.loads(l)
    print(d["config"], d["setting"], d["xwin"]["variant"], d["xwin"].get("ctas_per_sm"), d["xwin"]["cap_x"], d["xwin"].get("diag_warps"), d["xwin"].get("matrix_bytes"), round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()})
PY
grep -E "FAIL|Error|assert" gpurun_out/r62_xwin_pytest.log | head -30
