"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import re
import sys


def main(path, skip=0):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    body = [r for r in rows[hi + 1:] if len(r) > vi][skip:]
    for r in body:
        m = re.search(r"(k_\w+|at::\w+)", r[ki])
        name = m.group(1) if m else r[ki][:40]
        v = float(r[vi].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{'kernel':32s} {'launches':>8s} {'total_us':>10s} {'share':>6s} {'avg_us':>8s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:32s} {cnt[k]:8d} {v:10.1f} {100 * v / T:5.1f}% {v / cnt[k]:8.2f}")
    print(f"total {T:.1f} us over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
