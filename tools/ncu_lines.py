"""Per CUDA-source-line instruction and stall share of one kernel from an ncu report
(ncu --page source --print-source cuda,sass; needs -lineinfo).  Usage: ncu_lines.py REP KERNEL [N]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
if rep.endswith(".csv"):  # exported on the GPU box by tools/ncu_capture.sh (one kernel)
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
inst = defaultdict(float)
stall = defaultdict(float)
text = {}
fname = None
hdr = None
for r in csv.reader(raw.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: j for j, h in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    key = (fname, ln)
    text[key] = r[1].strip()[:90]
    try:
        inst[key] += float(r[hdr["Instructions Executed"]] or 0)
        stall[key] += float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, KeyError):
        pass
ti = sum(inst.values()) or 1
ts = sum(stall.values()) or 1
for key in sorted(inst, key=lambda k: -inst[k])[:top]:
    print(f"{key[0]}:{key[1]:<5d} inst {inst[key] / ti:6.3f} stall {stall[key] / ts:6.3f}  {text[key]}")
