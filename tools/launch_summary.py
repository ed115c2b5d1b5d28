"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def summary(path, top=10):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        k = r[ki].split("(")[0].replace("void unnamed>::", "").replace("void qoc::", "")
        agg[k][0] += 1
        agg[k][1] += float(r[vi].replace(",", "")) / 1e6
    tot = sum(v[1] for v in agg.values())
    out = [f"{path}: {len(rows)} launches, {tot:.2f} ms total (cold, serialised)"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"  {k:48s} n={v[0]:4d} {v[1]:9.3f} ms {100 * v[1] / tot:5.1f}%  {v[1] / v[0]:8.4f} ms/launch")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summary(p))
