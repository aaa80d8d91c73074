"""Per-kernel summary of an ncu --set full report (raw page): duration, pipes, DRAM, top stalls."""
import csv, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h = r[0]
units = dict(zip(h, r[1]))
for row in r[2:]:
    d = dict(zip(h, row))
    print(d['Kernel Name'][:60], '| grid', d.get('launch__grid_size'), '| block', d.get('launch__block_size'),
          '| duration', d.get('gpu__time_duration.sum'), units.get('gpu__time_duration.sum'),
          '| regs', d.get('launch__registers_per_thread'))
    for k in ['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
              'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
              'sm__throughput.avg.pct_of_peak_sustained_elapsed',
              'dram__bytes_read.sum', 'dram__bytes_write.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
              'lts__t_bytes.sum', 'smsp__warps_active.avg.per_cycle_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active']:
        if k in d: print('    %-70s %s %s' % (k, d[k], units.get(k, '')))
    st = [(k, float(v)) for k, v in d.items() if 'issue_stalled' in k and k.endswith('per_issue_active.ratio') and v]
    st.sort(key=lambda t: -t[1])
    print('    stalls/issue', [(k.split('stalled_')[1].split('_per')[0], round(v, 2)) for k, v in st[:8]])
