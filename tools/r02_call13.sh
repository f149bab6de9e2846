#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python tools/spmv_longrow_bench.py 4000000 auto 8 12 16 24 32 64 > gpurun_out/r13_longrow_sweep.jsonl 2>&1; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r13_longrow_sweep.jsonl"):
    try: d = json.loads(l)
    except Exception: print(l[:200]); continue
    print(d["threshold_env"], d["long_rows"], round(d["spmv_ms"], 4), round(d["frac"], 4), d["bitwise_vs_oracle"])
PY
