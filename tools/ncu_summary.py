"""Summarise an ncu --set full report: key throughput metrics + top stalls."""
import csv
import io
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed.avg.per_cycle_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'lts__t_bytes.sum', 'launch__grid_size',
        'launch__waves_per_multiprocessor', 'sm__cycles_elapsed.avg.per_second',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__inst_executed.sum']


def summarize(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        name = vals[hdr.index('Kernel Name')]
        lines = [f'kernel: {name[:110]}']
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                lines.append(f'  {w:68s} {vals[i]:>18s} {units[i]}')
        st = [(float(vals[i]), h) for i, h in enumerate(hdr)
              if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio')
              and vals[i] not in ('', 'n/a')]
        lines.append('  top stalls (warps per issue-active cycle):')
        for v, h in sorted(st, reverse=True)[:6]:
            lines.append(f'    {h[34:-27]:40s} {v:7.3f}')
        res.append('\n'.join(lines))
    return '\n'.join(res)


if __name__ == '__main__':
    for p in sys.argv[1:]:
        print(f'== {p}')
        print(summarize(p))
