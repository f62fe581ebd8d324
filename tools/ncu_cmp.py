"""Side-by-side key metrics of the first kernel in each .ncu-rep given."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum']
STALLS = ['short_scoreboard', 'mio_throttle', 'wait', 'math_pipe_throttle', 'barrier',
          'long_scoreboard', 'no_instruction', 'lg_throttle', 'dispatch_stall', 'not_selected',
          'branch_resolving', 'drain', 'sleeping', 'tex_throttle', 'imc_miss', 'misc']
WANT += ['smsp__average_warps_issue_stalled_%s_per_issue_active.ratio' % s for s in STALLS]


def load(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, d = r[0], r[2]
    return {w: d[h.index(w)] for w in WANT if w in h}


cols = [load(p) for p in sys.argv[1:]]
for w in WANT:
    vals = [c.get(w, '-') for c in cols]
    if all(v == '-' for v in vals):
        continue
    name = w.replace('smsp__average_warps_issue_stalled_', 'stall ').replace(
        '_per_issue_active.ratio', '')
    print('%-62s %s' % (name, '  '.join('%16s' % v for v in vals)))
