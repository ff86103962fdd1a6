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
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
mult = {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1}
path = 'profiles/traffic.json'
out = json.load(open(path)) if os.path.exists(path) else {}
if out and not all(isinstance(v, dict) and all(isinstance(x, dict) for x in v.values()) for v in out.values()):
    out = {}  # old flat layout (kernel -> figures) is replaced
ent = out.setdefault(cfg, {})
for r in rows[2:]:
    n = r[hdr.index('Kernel Name')].split('(')[0].split('<')[0].replace('void ', '').strip()
    b = sum(float(r[hdr.index(k)].replace(',', '')) * mult[units[hdr.index(k)]]
            for k in ['dram__bytes_read.sum', 'dram__bytes_write.sum'])

    def num(k):
        try:
            return float(r[hdr.index(k)].replace(',', ''))
        except (ValueError, IndexError):
            return None
    ent[n] = {"dram_bytes_per_launch": b, "source": f"{summary} (ncu --set full, 1 launch)",
              "version": tag,
              "issue_active_pct": num('smsp__issue_active.avg.pct_of_peak_sustained_active'),
              "active_threads_per_warp_inst": num('smsp__thread_inst_executed_per_inst_executed.ratio'),
              "warps_active_pct": num('sm__warps_active.avg.pct_of_peak_sustained_active'),
              "inst_executed_per_launch": num('smsp__inst_executed.sum'),
              "ncu_duration_ns": num('gpu__time_duration.sum'),
              "sm_mhz": num('sm__cycles_elapsed.avg.per_second')}
json.dump(out, open(path, 'w'), indent=1)
print(json.dumps(ent, indent=1))
