"""Merge the dram bytes per launch (and ncu limiter figures) of each kernel of one ncu report
into profiles/traffic.json under the report's config.
Usage: traffic_json.py REPORT TAG CONFIG [SUMMARY]   (SUMMARY: the committed profiles/ text file)"""
import csv
import json
import os
import subprocess
import sys

rep, tag, cfg = sys.argv[1], sys.argv[2], sys.argv[3]
summary = sys.argv[4] if len(sys.argv) > 4 else f"profiles/{tag}_ncu_{cfg}.txt"
if rep.endswith(".csv"):  # `ncu -i REP --page raw --csv` output written on the GPU box
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
mult = {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1}
path = 'profiles/traffic.json'
out = json.load(open(path)) if os.path.exists(path) else {}
if out and not all(isinstance(v, dict) and all(isinstance(x, dict) for x in v.values()) for v in out.values()):
    out = {}  # old flat layout (kernel -> figures) is replaced
ent = out.setdefault(cfg, {})
acc = {}
for r in rows[2:]:
    n = r[hdr.index('Kernel Name')].split('(')[0].split('<')[0].replace('void ', '').strip()
    b = sum(float(r[hdr.index(k)].replace(',', '')) * mult[units[hdr.index(k)]]
            for k in ['dram__bytes_read.sum', 'dram__bytes_write.sum'])

    def num(k):
        try:
            return float(r[hdr.index(k)].replace(',', ''))
        except (ValueError, IndexError):
            return None
    a = acc.setdefault(n, {"n": 0, "bytes": 0.0, "inst": 0.0, "issue": 0.0, "simt": 0.0, "warps": 0.0,
                           "dur": 0.0})
    a["n"] += 1
    a["bytes"] += b
    a["inst"] += num('smsp__inst_executed.sum') or 0.0
    a["issue"] += num('smsp__issue_active.avg.pct_of_peak_sustained_active') or 0.0
    a["simt"] += num('smsp__thread_inst_executed_per_inst_executed.ratio') or 0.0
    a["warps"] += num('sm__warps_active.avg.pct_of_peak_sustained_active') or 0.0
    a["dur"] += num('gpu__time_duration.sum') or 0.0
# per-launch averages over the captured launches of each kernel (launch-weighted)
for n, a in acc.items():
    k = a["n"]
    ent[n] = {"dram_bytes_per_launch": a["bytes"] / k, "source": f"{summary} (ncu --set full, {k} launch(es))",
              "version": tag, "issue_active_pct": a["issue"] / k, "active_threads_per_warp_inst": a["simt"] / k,
              "warps_active_pct": a["warps"] / k, "inst_executed_per_launch": a["inst"] / k,
              "ncu_duration_per_launch": a["dur"] / k, "launches": k}
json.dump(out, open(path, 'w'), indent=1)
print(json.dumps(ent, indent=1))
