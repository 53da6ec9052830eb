"""Print the key raw metrics of an ncu report: python tools/ncu_keys.py rep.ncu-rep"""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'smsp__warps_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active']
STALLS = ['barrier', 'long_scoreboard', 'short_scoreboard', 'wait', 'math_pipe_throttle',
          'mio_throttle', 'not_selected', 'selected', 'lg_throttle', 'dispatch_stall',
          'no_instructions', 'membar', 'sleeping', 'branch_resolving', 'drain', 'tex_throttle']
for rep in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print('==', rep, v[h.index('Kernel Name')][:80])
        for k in KEYS:
            if k in h:
                print(f'  {k:60s} {v[h.index(k)]:>14s} {u[h.index(k)]}')
        st = {s: v[h.index('smsp__pcsamp_warps_issue_stalled_' + s)] for s in STALLS
              if 'smsp__pcsamp_warps_issue_stalled_' + s in h}
        print('  stalls:', ' '.join(f'{k}={x}' for k, x in st.items() if x not in ('0', '')))
