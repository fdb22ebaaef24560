"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def summarize(path, top=15):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}.get(r[ui], 1)
        name = r[ki].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    out = [f"total kernel time {T / 1e3:.3f} ms", "", "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        out.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / T:.1f}% |")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        print(summarize(p))
