"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count and total time."""
import csv
import sys
from collections import defaultdict


def summarise(path, top=30):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) > iv:
            k = r[ik].split("(")[0][:70]
            agg[k][0] += 1
            agg[k][1] += float(r[iv].replace(",", ""))
    total = sum(t for _, t in agg.values())
    out = []
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{c:4d} {t / 1e3:10.1f} us {100 * t / total:5.1f}%  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
