"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
per-kernel count, total and mean device time, share of the total."""
import collections
import csv
import sys


def summarize(path, skip_prefix=("<unnamed>::k_fill", "h2d::k_deinterleave", "h2d::k_interleave")):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in rows if r[0] == "ID")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[rows.index(hdr) + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        if name.startswith(skip_prefix):
            continue
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1.0)
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':48s} {'n':>4s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k:48s} {n:4d} {t:10.1f} {t / n:9.2f} {t / tot:6.3f}")
    out.append(f"{'TOTAL':48s} {'':4s} {tot:10.1f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
