"""Summarise an ncu launch-list CSV (gpu__time_duration.sum) per kernel."""
import collections, csv, sys

def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    out = []
    for r in data:
        out.append((r[ki].split("(")[0], float(r[vi].replace(",", "")) * scale[r[ui]]))
    return out

if __name__ == "__main__":
    launches = load(sys.argv[1])
    only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, us in launches:
        if only and not any(o in name for o in only):
            continue
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'n':>5s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:60]:60s} {c:5d} {t:10.1f} {t / c:9.2f} {t / tot:6.3f}")
