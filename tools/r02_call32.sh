#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_dia.py -q --timeout 300 -p no:cacheprovider > gpurun_out/r70_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r70_pytest.log
for pf in 1 0; do
SPARSLA_DIA_PREFETCH=$pf timeout 600 python tools/xw_sweep.py B D > gpurun_out/r70_sweep_$pf.jsonl 2>/dev/null
python - $pf <<'PY'
import json, sys
for l in open(f"gpurun_out/r70_sweep_{sys.argv[1]}.jsonl"):
    d = json.loads(l)
    if d["setting"] in ("default", "xwin-1"):
        print("prefetch", sys.argv[1], d["config"], d["setting"], round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()})
PY
done
