"""All 'details' page metrics of the sections that explain a latency-bound kernel.
usage: python tools/ncu_details.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get('Section Name') in ('Compute Workload Analysis', 'Memory Workload Analysis', 'Scheduler Statistics',
                                 'Warp State Statistics', 'Instruction Statistics', 'Memory Workload Analysis Tables',
                                 'Shared Memory'):
        print(f"{d['Section Name'][:28]:28s} {d['Metric Name']:52s} {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    h, v = rr[0], rr[2]
    for i, k in enumerate(h):
        if any(t in k for t in ('pipe_', 'l1tex__data_bank_conflicts', 'shared_ld', 'shared_st', 'shared_atom', 'data_pipe_lsu_wavefronts_mem_shared',
                                'smsp__warp_issue_stalled', 'inst_executed_op_shared')):
            print(f"{k:90s} {v[i]}")
