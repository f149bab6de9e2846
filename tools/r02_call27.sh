#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python tools/xw_sweep.py B D --variants=12 > gpurun_out/r64_xw_sweep.jsonl 2> gpurun_out/r64_xw_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r64_xw_sweep.jsonl"):
    d = json.loads(l)
    print(d["config"], d["setting"], d["xwin"]["variant"], d["xwin"].get("diag_warps"), round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()})
PY
