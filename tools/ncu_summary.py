"""Print the key metrics + top stall reasons of every kernel in an ncu report (or its raw-page
CSV export)."""
import csv
import subprocess
import sys

if sys.argv[1].endswith(".csv"):  # raw page exported on the GPU box (tools/ncu_capture.sh)
    raw = open(sys.argv[1]).read()
else:
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'smsp__inst_executed.sum', 'l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum', 'l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum',
        'lts__t_bytes.sum']
for r in rows[2:]:
    print('##', r[hdr.index('Kernel Name')].split('(')[0])
    for k in keys:
        if k in hdr:
            print(f'  {k:58s} {r[hdr.index(k)]} {units[hdr.index(k)]}')
    st = []
    for i, h in enumerate(hdr):
        if h.startswith('smsp__pcsamp_warps_issue_stalled') and 'not_issued' not in h:
            try:
                st.append((float(r[i].replace(',', '')), h.replace('smsp__pcsamp_warps_issue_stalled_', '')))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print('  stalls:', ', '.join(f'{n} {v / tot:.2f}' for v, n in sorted(st, reverse=True)[:7]))
