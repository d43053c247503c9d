"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram/lts bytes]) per kernel.

    python profiles/summarize_launches.py gpurun_out/launches.csv
"""
import collections
import csv
import sys

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, ii, mi, ui, vi = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Unit", "Metric Value"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("isvd::<unnamed>::", "").replace("void ", "")
    return per, names


def main():
    per, names = load(sys.argv[1])
    tot = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for i, m in per.items():
        k = names[i]
        cnt[k] += 1
        for mn, v in m.items():
            tot[k][mn] += v
    T = sum(t["gpu__time_duration.sum"] for t in tot.values())
    print(f"{'kernel':44s} {'n':>5s} {'total ms':>10s} {'share':>6s} {'avg us':>10s} {'DRAM GB/s':>10s} {'DRAM MB/launch':>14s}")
    for k, t in sorted(tot.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        us = t["gpu__time_duration.sum"]
        dram = t.get("dram__bytes_read.sum", 0) + t.get("dram__bytes_write.sum", 0)
        bw = dram / (us * 1e-6) / 1e9 if us else 0
        print(f"{k[:44]:44s} {cnt[k]:5d} {us/1e3:10.2f} {100*us/T:5.1f}% {us/cnt[k]:10.1f} {bw:10.0f} {dram/cnt[k]/1e6:14.1f}")
    print(f"total {T/1e3:.2f} ms over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main()
