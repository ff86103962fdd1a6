"""Per-region instruction share / stall share / active threads from an ncu SASS source page."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
W = int(sys.argv[3]) if len(sys.argv) > 3 else 48
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[1]
ci = {h: j for j, h in enumerate(hdr)}
seen, out = set(), []
for r in rows[2:]:
    try:
        a = int(r[ci['Address']], 16)
    except (ValueError, KeyError, IndexError):
        continue
    if a in seen:
        continue
    seen.add(a)
    f = lambda k: float(r[ci[k]] or 0)
    out.append((a, r[ci['Source']].strip(), f('Instructions Executed'), f('Thread Instructions Executed'),
                f('Warp Stall Sampling (All Samples)')))
out.sort()
base = out[0][0]
ti = sum(o[2] for o in out) or 1
ts = sum(o[4] for o in out) or 1
for k in range(0, len(out), W):
    seg = out[k:k + W]
    ie = sum(o[2] for o in seg)
    if ie / ti < 0.01:
        continue
    te = sum(o[3] for o in seg)
    s = sum(o[4] for o in seg)
    kinds = {}
    for o in seg:
        op = (o[1].split()[1] if o[1].startswith('@') else o[1].split()[0]).split('.')[0]
        kinds[op] = kinds.get(op, 0) + 1
    top = ','.join(f"{a}{b}" for a, b in sorted(kinds.items(), key=lambda x: -x[1])[:6])
    print(f"{hex(seg[0][0] - base):>7s} inst {ie / ti:5.3f} stall {s / ts:5.3f} thr/inst {te / max(ie, 1):5.1f}  {top}")
