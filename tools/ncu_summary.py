"""Summarise an ncu --set full report (raw page) into a short text block per
kernel launch: time, DRAM bytes, instructions, issue / occupancy, top stalls.

    python tools/ncu_summary.py report.ncu-rep [title]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__shared_mem_per_block_static", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(title)
    for v in rows[2:]:
        d = dict(zip(hdr, v))
        un = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name', '?')}  grid {d.get('Grid Size', '')} block {d.get('Block Size', '')}")
        for k in KEYS:
            if k in d:
                print(f"  {k:62s} {d[k]} {un.get(k, '')}")
        st = [k for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and
              k.endswith("_per_issue_active.ratio")]
        vals = sorted(((float(d[k].replace(",", "")), k) for k in st if d[k] not in ("", "n/a")), reverse=True)[:6]
        print("  stalls (cycles per issued instruction): " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {x:.2f}"
            for x, k in vals))


if __name__ == "__main__":
    main()
