"""Summarise an .ncu-rep: key raw metrics + stall breakdown + hottest SASS lines."""
import csv, subprocess, sys, io

def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]

KEYS = ['Kernel Name', 'gpu__time_duration.sum', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'l1tex__t_bytes.sum',
        'sm__cycles_elapsed.avg', 'smsp__cycles_active.avg']

def main(rep, nsass=40):
    hdr, units, rows = raw(rep)
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows:
        print('-----')
        for k in KEYS:
            if k in idx:
                print(f'  {k} = {r[idx[k]]} {units[idx[k]]}')
        st = [(h, float(r[i])) for h, i in idx.items()
              if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio')
              and r[i] not in ('', 'n/a')]
        st.sort(key=lambda t: -t[1])
        print('  stalls/issue:', ', '.join(f"{h.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')}={v:.2f}" for h, v in st[:8]))

if __name__ == '__main__':
    main(sys.argv[1])
