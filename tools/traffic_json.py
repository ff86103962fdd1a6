"""Write profiles/traffic.json (dram bytes per launch of each kernel) from an ncu report."""
import csv
import json
import subprocess
import sys

rep, tag = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
mult = {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1}
out = {}
for r in rows[2:]:
    n = r[hdr.index('Kernel Name')].split('(')[0]
    b = sum(float(r[hdr.index(k)].replace(',', '')) * mult[units[hdr.index(k)]]
            for k in ['dram__bytes_read.sum', 'dram__bytes_write.sum'])
    def num(k):
        try:
            return float(r[hdr.index(k)].replace(',', ''))
        except (ValueError, IndexError):
            return None
    out[n] = {"dram_bytes_per_launch": b, "source": f"profiles/{tag}_ncu_trace.txt (ncu --set full, 1 launch)",
              "version": tag,
              "issue_active_pct": num('smsp__issue_active.avg.pct_of_peak_sustained_active'),
              "active_threads_per_warp_inst": num('smsp__thread_inst_executed_per_inst_executed.ratio'),
              "warps_active_pct": num('sm__warps_active.avg.pct_of_peak_sustained_active')}
json.dump(out, open('profiles/traffic.json', 'w'), indent=1)
print(out)
