"""Stall samples and executed instructions of one kernel aggregated by CUDA
source line (ncu report, source page with cuda+sass correlation):
python tools/src_hot.py report.ncu-rep kernel_regex [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
samp = collections.Counter()
inst = collections.Counter()
text = {}
fname = "?"
cur = None
tot_s = tot_i = 0
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a source line row
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()[:90]
        continue
    if r[2] in ("...", "-") or cur is None:
        continue
    try:
        s = int(r[4]); n = int(r[7])
    except ValueError:
        continue
    samp[cur] += s
    inst[cur] += n
    tot_s += s
    tot_i += n
print(f"{kern}: {tot_s} samples, {tot_i/1e6:.1f} M warp-inst (sass rows may repeat per inlined site)")
for k, s in samp.most_common(top):
    print(f"{100*s/tot_s:5.1f}% smp {100*inst[k]/max(tot_i,1):5.1f}% inst  {k[0]}:{k[1]}  {text.get(k,'')}")
