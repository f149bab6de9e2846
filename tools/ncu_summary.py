"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    H = rows[hdr]
    ki, mi, vi = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].split("::")[-1][:44]
        agg[name][r[mi]] += float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            cnt[name] += 1
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    print(f"{'kernel':44s} {'launches':>8s} {'total ms':>9s} {'share':>6s} {'avg us':>8s} {'DRAM GB/s':>9s}")
    for n, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        t = a["gpu__time_duration.sum"]
        b = a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)
        print(f"{n:44s} {cnt[n]:8d} {t / 1e6:9.3f} {t / tot:6.1%} {t / cnt[n] / 1e3:8.1f} {b / t if t else 0:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
