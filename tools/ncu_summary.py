"""Summarise an ncu report: key SOL/occupancy/scheduler metrics + hot SASS buckets."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
keys = ('GPU Speed Of Light Throughput', 'Occupancy', 'Compute Workload Analysis',
        'Memory Workload Analysis', 'Scheduler Statistics', 'Warp State Statistics', 'Launch Statistics')
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = ('Duration', 'Elapsed Cycles', 'DRAM Throughput', 'Compute (SM) Throughput', 'Executed Ipc Active',
        'Issue Slots Busy', 'Achieved Active Warps Per SM', 'Theoretical Active Warps per SM',
        'Registers Per Thread', 'Dynamic Shared Memory Per Block', 'Grid Size', 'Block Size',
        'Eligible Warps Per Scheduler', 'No Eligible', 'Warp Cycles Per Issued Instruction',
        'L1/TEX Cache Throughput', 'L2 Cache Throughput', 'Mem Busy', 'Waves Per SM')
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get('Section Name') in keys and d.get('Metric Name') in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    h, v = rr[0], rr[2]
    for name in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
                 'sm__inst_executed_pipe_lsu.sum', 'smsp__average_warp_latency_issue_stalled_short_scoreboard'):
        for i, k in enumerate(h):
            if k.startswith(name):
                print(f"{k:60s} {v[i]}")
sass = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=sass'],
                      capture_output=True, text=True).stdout
sr = list(csv.reader(io.StringIO(sass)))
if len(sr) > 2:
    h = sr[1]
    data = sr[2:]
    ie = h.index('Instructions Executed')
    smp = h.index('Warp Stall Sampling (All Samples)')
    st = {k: h.index(k) for k in h if k.startswith('stall_') and '(Not Issued)' not in k}
    tot = {k: sum(int(r[i] or 0) for r in data) for k, i in st.items()}
    s = sum(tot.values()) or 1
    print('stall breakdown:', ', '.join(f"{k[6:]}={100*v/s:.0f}%" for k, v in sorted(tot.items(), key=lambda t: -t[1])[:8]))
    print('total warp instr:', sum(int(r[ie] or 0) for r in data))
