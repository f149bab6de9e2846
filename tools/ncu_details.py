"""Print key ncu --set full metrics + top stall reasons per captured kernel (ncu -i REP)."""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Grid Size", "Block Size", "L2 Hit Rate", "L1/TEX Hit Rate"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    ki, ni, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    cur = None
    for x in r[1:]:
        if x[ni] in WANT:
            if x[ii] != cur:
                cur = x[ii]
                print(f"--- {x[ii]} {x[ki][:60]}")
            print(f"   {x[ni]:28s} {x[vi]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h = r[0]
    for row in r[2:]:
        d = dict(zip(h, row))
        st = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    st.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", ""))))
                except ValueError:
                    pass
        st.sort(key=lambda t: -t[1])
        tot = sum(v for _, v in st) or 1
        print(d.get("ID"), d["Kernel Name"][:40], " ".join(f"{k}:{v / tot:.0%}" for k, v in st[:5]))


if __name__ == "__main__":
    main(sys.argv[1])
