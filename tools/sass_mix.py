"""Opcode mix and stall samples of one kernel from an ncu report's SASS
source page: python tools/sass_mix.py report.ncu-rep kernel_regex"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: k for k, h in enumerate(hdr)}
inst = collections.Counter()
samp = collections.Counter()
tot_i = tot_s = 0
for r in rows[2:]:
    if len(r) < len(hdr) or not r[ix["Source"]].strip() or r[ix["Source"]] == "Source":
        continue
    op = r[ix["Source"]].split()[0]
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    op = op.split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    inst[op] += n
    samp[op] += s
    tot_i += n
    tot_s += s
print(f"{kern}: {tot_i/1e6:.1f} M warp-instructions, {tot_s} stall samples")
for op, n in inst.most_common(28):
    print(f"  {op:10s} {100*n/tot_i:5.1f}% inst  {100*samp[op]/max(tot_s,1):5.1f}% samples")
