"""Summarise an ncu --set full report (raw page) for the roofline: time, DRAM bytes, key throughputs, stalls."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__m_l1tex2xbar_write_bytes_mem_global_op_tma_red.sum.pct_of_peak_sustained_elapsed',
        'sm__cycles_elapsed.avg.per_second', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active']


def summary(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        name = r[h.index('Kernel Name')] if 'Kernel Name' in h else '?'
        lines = [f'kernel: {name[:110]}']
        for i, k in enumerate(h):
            if k in WANT:
                lines.append(f'  {k:78s} {r[i]:>16s} {u[i]}')
        st = []
        for i, k in enumerate(h):
            if 'average_warps_issue_stalled' in k and k.endswith('per_issue_active.ratio'):
                try:
                    st.append((float(r[i]), k.replace('smsp__average_warps_issue_stalled_', '').replace(
                        '_per_issue_active.ratio', '')))
                except ValueError:
                    pass
        lines.append('  top stalls (warps per issue): ' + ', '.join(f'{n}={v:.2f}' for v, n in sorted(st)[::-1][:5]))
        res.append('\n'.join(lines))
    return '\n'.join(res)


if __name__ == '__main__':
    for p in sys.argv[1:]:
        print(f'== {p}')
        print(summary(p))
