"""Quick per-kernel readout of an ncu report: duration, issue, pipes, L1/L2, top stalls.

    python tools/ncu_quick.py gpurun_out/x.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'smsp__issue_active.avg.per_cycle_active',
        'smsp__warps_active.avg.per_cycle_active', 'launch__registers_per_thread',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'l1tex__t_sector_hit_rate.pct',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'dram__bytes_read.sum', 'dram__bytes_write.sum']
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
for v in rows[2:]:
    print('==', v[h.index('Kernel Name')][:90])
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f'  {k:62s} {v[i]:>16s} {u[i]}')
    st = sorted(((float(v[i]), n[34:-23]) for i, n in enumerate(h)
                 if n.startswith('smsp__average_warps_issue_stalled_') and n.endswith('_per_issue_active.ratio')), reverse=True)
    print('  stalls:', ', '.join(f'{n} {x:.2f}' for x, n in st[:5]))
