"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel count,
total device time and share (ncu serialises and cold-starts every launch: compare SHARES)."""
import collections
import csv
import sys


def summarize(path):
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
        name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':40s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k[:40]:40s} {n:8d} {t:12.1f} {t / n:10.1f} {t / tot:7.3f}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
