"""Per-kernel table from an ncu --csv launch list with time, DRAM bytes,
occupancy, fp64-pipe and instruction metrics (means over launches)."""
import collections
import csv
import sys

SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def table(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in rows if r[0] == "ID")
    data, names = collections.defaultdict(dict), {}
    for r in rows[rows.index(hdr) + 1:]:
        d = dict(zip(hdr, r))
        data[d["ID"]][d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
        names[d["ID"]] = d["Kernel Name"].split("(")[0]
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    for i, m in data.items():
        a = agg[names[i]]
        a["n"] += 1
        t = m["gpu__time_duration.sum"]
        a["us"] += t[0] * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(t[1], 1.0)
        for k, key in (("R", "dram__bytes_read.sum"), ("W", "dram__bytes_write.sum")):
            if key in m:
                a[k] += m[key][0] * SC.get(m[key][1], 1)
        for k, key in (("occ", "sm__warps_active.avg.pct_of_peak_sustained_active"),
                       ("fp64", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                       ("inst", "smsp__inst_executed.sum")):
            if key in m:
                a[k] += m[key][0]
    out = [f"{'kernel':34s} {'n':>3s} {'mean_us':>8s} {'R_MB':>7s} {'W_MB':>7s} {'GB/s':>6s} {'occ%':>5s} {'fp64%':>6s} {'Minst':>7s}"]
    tot = sum(a["us"] for a in agg.values())
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        n = a["n"]
        out.append(f"{k:34s} {int(n):3d} {a['us'] / n:8.1f} {a['R'] / n / 1e6:7.1f} {a['W'] / n / 1e6:7.1f} "
                   f"{(a['R'] + a['W']) / a['us'] / 1e3:6.0f} {a['occ'] / n:5.1f} {a['fp64'] / n:6.1f} "
                   f"{a['inst'] / n / 1e6:7.2f}")
    out.append(f"total {tot:.1f} us over all launches")
    return "\n".join(out)


if __name__ == "__main__":
    print(table(sys.argv[1]))
