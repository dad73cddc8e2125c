"""Aggregate an ncu --metrics gpu__time_duration.sum CSV by kernel."""
import collections
import csv
import re
import sys


def main(path, top=16):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h, rows = rows[0], rows[1:]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = re.sub(r"\(.*", "", r[ik]).replace("unnamed>::", "")
        val = float(r[iv].replace(",", ""))
        val *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[iu], 1.0)
        agg[name][0] += 1
        agg[name][1] += val
    tot = sum(v[1] for v in agg.values())
    print(f"launches {len(rows)}, summed kernel time {tot / 1e6:.3f} ms (cold-cache, serialised by ncu)")
    print(f"{'ms':>10} {'share':>6} {'count':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v[1] / 1e6:10.3f} {100 * v[1] / tot:5.1f}% {v[0]:6d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
