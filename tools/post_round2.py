"""Turn a measurement set brought back in gpurun_out/ (tools/prof_round2b.sh)
into the committed files under profiles/: bench lines, launch tables (text +
csv), ncu --set full summaries, and profiles/traffic_per_launch.json (the
per-launch DRAM bytes bench.py reports as roofline.traffic).

    python tools/post_round2.py v2
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import launch_summary  # noqa: E402
import launch_table  # noqa: E402

V = sys.argv[1] if len(sys.argv) > 1 else "v2"
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
KERNELS = ("k_lag_fused", "k_remap_tile", "k_dual_items", "k_node_update_walls", "k_post")


def traffic(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in rows if r[0] == "ID")
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in rows[rows.index(hdr) + 1:]:
        d = dict(zip(hdr, r))
        if d["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            per[(d["ID"], d["Kernel Name"].split("(")[0])]["b"] += float(d["Metric Value"].replace(",", "")) * \
                SC.get(d["Metric Unit"], 1)
    agg = collections.defaultdict(list)
    for (_, name), v in per.items():
        for k in KERNELS:
            if k in name:
                agg[k].append(v["b"])
    return {k: int(sum(v) / len(v)) for k, v in agg.items() if v}


def main():
    for f in sorted(os.listdir(G)):
        if f.startswith("r02_bench_") and f.endswith(f"_{V}.json") and os.path.getsize(os.path.join(G, f)) > 0:
            shutil.copy(os.path.join(G, f), os.path.join(P, f))
    if os.path.exists(os.path.join(G, f"r02_box_{V}.txt")):
        shutil.copy(os.path.join(G, f"r02_box_{V}.txt"), os.path.join(P, f"r02_box_{V}.txt"))
    tr = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch (mean over launches), ncu "
                   "--clock-control none, cold caches; c5b = one 4096x8192 block of the 16384^2 mesh",
          "_source": f"profiles/r02_*_launches_{V}.csv"}
    for wl in ("c4", "c2", "c5b"):
        src = os.path.join(G, f"r02_{wl}_launches_{V}.csv")
        if not os.path.exists(src) or os.path.getsize(src) == 0:
            continue
        shutil.copy(src, os.path.join(P, os.path.basename(src)))
        with open(os.path.join(P, f"r02_{wl}_launches_{V}.txt"), "w") as f:
            f.write(launch_table.table(src) + "\n")
        t = traffic(src)
        t["_source"] = f"profiles/r02_{wl}_launches_{V}.csv"
        tr[wl] = t
    if len(tr) > 2:
        with open(os.path.join(P, "traffic_per_launch.json"), "w") as f:
            json.dump(tr, f, indent=1)
    src = os.path.join(G, f"r02_bench_launches_{V}.csv")
    if os.path.exists(src) and os.path.getsize(src) > 0:
        shutil.copy(src, os.path.join(P, os.path.basename(src)))
        with open(os.path.join(P, f"r02_bench_launches_{V}.txt"), "w") as f:
            f.write(launch_summary.summarize(src) + "\n")
    for wl in ("c4", "c5b"):
        rep = os.path.join(G, f"r02_{wl}_full_{V}.ncu-rep")
        if os.path.exists(rep):
            out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep,
                                  f"gpurun_out/r02_{wl}_full_{V}.ncu-rep"], capture_output=True, text=True).stdout
            with open(os.path.join(P, f"r02_{wl}_full_{V}.txt"), "w") as f:
                f.write(out)


if __name__ == "__main__":
    main()
