"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import collections
import csv
import sys


def summarise(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
        name = r[ki].split("(")[0][:70]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    out = []
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        out.append(f"{v / 1e6:9.3f} ms {100 * v / T:5.1f}% n={cnt[k]:5d} avg={v / cnt[k] / 1e3:8.1f}us {k}")
    out.append(f"total ms {T / 1e6:.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25))
