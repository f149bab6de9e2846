#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python tools/xw_sweep.py B E D > gpurun_out/r51_xw_sweep.jsonl 2> gpurun_out/r51_xw_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r51_xw_sweep.jsonl"):
    d = json.loads(l)
    if "plain" in d["setting"]: continue
    print(d["config"], d["setting"], d["xwin"]["variant"], round(d["iteration_ms"], 4), {k: round(v, 4) for k, v in d["ms"].items()})
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:spmv_xw -s 3 -c 2 --csv python tools/spmv_profile.py poisson3d 464 cg 2>/dev/null | grep spmv_xw | awk -F'","' '{print $(NF-2) " " $NF}'
