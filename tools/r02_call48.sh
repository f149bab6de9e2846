#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "long_rows or hub or direct or random" --timeout 600 -p no:cacheprovider > gpurun_out/r48_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r48_pytest.log | tail -3
timeout 1200 python tools/spmv_longrow_bench.py 4000000 auto 0 > gpurun_out/r48_longrow.jsonl 2>&1; echo "longrow rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r48_longrow.jsonl"):
    try: d = json.loads(l)
    except Exception: print(l[:200]); continue
    print(d["threshold_env"], d["long_rows"], round(d["spmv_ms"], 4), round(d["frac"], 4), d["bitwise_vs_oracle"])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r48_longrow_launches.csv python tools/spmv_longrow_bench.py 4000000 auto > /dev/null 2>&1; echo "ncu rc=$?"
